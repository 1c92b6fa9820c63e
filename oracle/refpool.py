"""The reference's own CPU decoder, run from its offline install -- TEST /
BASELINE INFRASTRUCTURE (like the rest of oracle/).

`bench.py --impl reference` and the CPU legs of the GPU arm time the
UNMODIFIED reference package (`ldpc_ids`, installed once into baseline/_ref
with pip --no-index; it travels to the GPU box with the repo snapshot) through
its public `schedules.decode` (schedules.py:111-158), fanned out over frame
blocks with a ProcessPoolExecutor exactly like the reference harness does
(sim.py:233-259, `_worker_init` + per-block `_sim_block`).  Numba's JIT is
warmed in each worker's initializer, so compile time stays outside the timed
region; NUMBA_CACHE_DIR points at a writable directory because the package
uses `@njit(cache=True)`.

The reference has no layered or ME-RBP schedule (schedules.py:20-21); those
two are reported as unavailable here (the C port in ldpc_oracle.c defines them).
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"
REF_KINDS = ("flooding", "rbp", "cirbp", "lmdrbp", "slmdrbp", "lmd_cirbp", "me_cirbp", "me_lmd_cirbp")

_W = {}


def available():
    return (REF_DIR / "ldpc_ids" / "schedules.py").exists()


def _import_ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ldpc_ids_numba_cache")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    from ldpc_ids import codes, schedules  # noqa: F401
    return codes, schedules


def _init(entries, m_rows, n_cols, punctured, k_info, label, scheds):
    rc, rs = _import_ref()
    h = rc.ParityCheckMatrix(m_rows=m_rows, n_cols=n_cols, entries=entries)
    spec = rc.CodeSpec(h=h, punctured=punctured, k_info=k_info, label=label)
    _W["spec"], _W["graph"], _W["rs"] = spec, rc.build_tanner(h), rs
    # JIT warm-up: one tiny decode per schedule (budget 1 iteration)
    z = np.full(n_cols, 2.0)
    for kind, n_p, i_max in scheds:
        rs.decode(spec, z, rs.ScheduleConfig(kind=kind, n_p=n_p, i_max=1), graph=_W["graph"])


def _ready(_):
    time.sleep(0.2)
    return os.getpid()


def _block(task):
    kind, n_p, i_max, llrs = task
    rs = _W["rs"]
    cfg = rs.ScheduleConfig(kind=kind, n_p=n_p, i_max=i_max)
    upd = fe = 0
    props, uh = [], []
    for row in llrs:
        r = rs.decode(_W["spec"], row, cfg, graph=_W["graph"])
        p = int(r.iterations_used * _W["graph"].n_edges)
        upd += p
        fe += int(r.bit_errors_at[i_max] > 0)
        props.append(p)
        uh.append(np.packbits(r.u_hat))
    return upd, fe, props, uh


class RefPool:
    """Worker pool holding the reference code + graph, JIT-warm."""

    def __init__(self, spec, scheds, i_max, workers=None):
        self.workers = workers or os.cpu_count() or 1
        self.scheds = [(k, n) for k, n in scheds if k in REF_KINDS]
        h = spec.h
        self.pool = ProcessPoolExecutor(
            max_workers=self.workers, initializer=_init,
            initargs=(h.entries, h.m_rows, h.n_cols, spec.punctured, spec.k_info, spec.label,
                      [(k, n, i_max) for k, n in self.scheds]))
        self.i_max = i_max
        # start every worker (initializer + JIT) before anything is timed
        list(self.pool.map(_ready, range(2 * self.workers)))

    def run(self, llrs):
        """Decode llrs[B, N] with every reference schedule; returns per-schedule
        (updates, frame errors, props, packed u_hat) and the wall time."""
        llrs = np.asarray(llrs, np.float64)
        nb = max(1, min(len(llrs), self.workers))
        blocks = np.array_split(np.arange(len(llrs)), nb)
        t0 = time.perf_counter()
        futs = {}
        for kind, n_p in self.scheds:
            futs[(kind, n_p)] = [self.pool.submit(_block, (kind, n_p, self.i_max, llrs[b])) for b in blocks if len(b)]
        out = {}
        for key, fl in futs.items():
            rs = [f.result() for f in fl]
            out[key] = (sum(r[0] for r in rs), sum(r[1] for r in rs),
                        np.array([p for r in rs for p in r[2]], np.int64), [u for r in rs for u in r[3]])
        return out, time.perf_counter() - t0

    def close(self):
        self.pool.shutdown(wait=True, cancel_futures=True)
