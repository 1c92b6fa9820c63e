"""Multi-GPU plumbing for batched decoding.

Frames are independent, so N GPUs decode disjoint frame shards with the graph
replicated and no data-path collective (weak scaling: each rank owns
`per_rank` consecutive frame indices, so the Philox frame substreams --
channel.py:71-74 -- never overlap).  The only collectives reduce the int64
tallies (frame/bit errors, C2V updates, counters) and the timing (max over
ranks) at the end, over NCCL on GPUs or gloo on CPUs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(per_rank: int, rank: int | None = None) -> tuple[int, int]:
    """(first frame index, count) of this rank's shard under weak scaling."""
    if rank is None:
        rank = world()[0]
    return rank * per_rank, per_rank


def _device():
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_sum(values) -> np.ndarray:
    """Element-wise sum over ranks of an int64 vector."""
    t = torch.as_tensor(np.asarray(values, dtype=np.int64), device=_device())
    if world()[1] > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def all_max(values) -> np.ndarray:
    """Element-wise max over ranks of a float64 vector (timings)."""
    t = torch.as_tensor(np.asarray(values, dtype=np.float64), device=_device())
    if world()[1] > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


@dataclass
class Tally:
    """Per-cell aggregates in the reference harness's sense (sim.py:146-171)."""

    i_max: int
    frames: int = 0
    frame_errors: int = 0       # bit_errors_at[i_max] > 0 over all N (sim.py:152-154)
    bit_errors: int = 0         # info bits (E:200-201)
    converged: int = 0
    propagations: int = 0
    counters: np.ndarray = field(default_factory=lambda: np.zeros(8, np.int64))
    frame_errors_at: np.ndarray = None
    bit_errors_at: np.ndarray = None

    def __post_init__(self):
        if self.frame_errors_at is None:
            self.frame_errors_at = np.zeros(self.i_max + 1, np.int64)
            self.bit_errors_at = np.zeros(self.i_max + 1, np.int64)

    def add(self, r):
        """Fold a results_to_numpy() dict (or oracle batch dict) in."""
        be = np.asarray(r["bit_errors_at"])
        bi = np.asarray(r["info_bit_errors_at"])
        self.frames += len(be)
        self.frame_errors += int((be[:, self.i_max] > 0).sum())
        self.bit_errors += int(bi[:, self.i_max].sum())
        self.converged += int(np.asarray(r["converged"]).sum())
        self.propagations += int(np.asarray(r["prop"]).sum())
        self.counters += np.asarray(r["counters"]).sum(0).astype(np.int64)
        self.frame_errors_at += (be > 0).sum(0)
        self.bit_errors_at += bi.sum(0)
        return self

    def _vec(self):
        return np.concatenate([[self.frames, self.frame_errors, self.bit_errors, self.converged,
                                self.propagations], self.counters, self.frame_errors_at,
                               self.bit_errors_at]).astype(np.int64)

    def reduce(self):
        """Sum over ranks (one all_reduce of a flat int64 vector)."""
        v = all_sum(self._vec())
        t = Tally(self.i_max)
        t.frames, t.frame_errors, t.bit_errors, t.converged, t.propagations = (int(x) for x in v[:5])
        t.counters = v[5:13]
        t.frame_errors_at = v[13:14 + self.i_max]
        t.bit_errors_at = v[14 + self.i_max:]
        return t

    @property
    def fer(self):
        return self.frame_errors / max(1, self.frames)
