"""Counters and kernel names (mirrors /root/reference/pkg/src/ldpc_ids/kernels.py:18-55)."""

from __future__ import annotations

from dataclasses import dataclass

LLR_MAX = 30.0
KERNELS = {"exact": 0, "minsum": 1}

COUNTER_NAMES = ("c2v_propagations", "v2c_updates", "c2v_pre_updates", "ci_updates",
                 "residual_ci_comparisons", "multi_select_comparisons", "kappa_hits",
                 "kappa_trials")


@dataclass
class Counters:
    c2v_propagations: int = 0
    v2c_updates: int = 0
    c2v_pre_updates: int = 0
    ci_updates: int = 0
    residual_ci_comparisons: int = 0
    multi_select_comparisons: int = 0
    kappa_hits: int = 0
    kappa_trials: int = 0

    @classmethod
    def from_array(cls, a):
        return cls(**{k: int(a[i]) for i, k in enumerate(COUNTER_NAMES)})

    def as_dict(self):
        return {k: getattr(self, k) for k in COUNTER_NAMES}
