"""Shared test helpers (no GPU, no reference import)."""

import ast
import functools
from pathlib import Path

import numpy as np

from paper_2102_11089_b200 import configs
from paper_2102_11089_b200.codes import build_tanner

GOLDEN = Path(__file__).resolve().parent / "golden"
FILES = {"c0": "C0", "c1": "C1", "c2": "C2", "c3": "C3", "c3b": "C3"}


@functools.lru_cache(maxsize=None)
def load_code(key):
    spec = {"C0": configs.make_c0_code, "C1": configs.make_c1_code, "C2": configs.make_c2_code,
            "C3": configs.make_c3_code}[key]()
    return spec, build_tanner(spec.h)


def golden_cases(files=("c0", "c1", "c2", "c3", "c3b")):
    out = []
    for f in files:
        z = np.load(GOLDEN / f"{f}.npz")
        for si, s in enumerate(z["schedules"]):
            out.append((f, FILES[f], si, ast.literal_eval(str(s))))
    return out


def golden_digest_ok(fname, g):
    z = np.load(GOLDEN / f"{fname}.npz")
    d = np.array([g.n_vars, g.n_checks, g.n_edges,
                  int(np.sum(g.edge_cn * 1_000_003 + g.edge_vn * 7) % (1 << 61))], np.int64)
    return bool((z["digest"] == d).all())


def p0_vec(llrs):
    """Stable logistic P(bit = 0) (kernels.posterior_p0 / sim._p0_vec, sim.py:186-192)."""
    llrs = np.asarray(llrs, np.float64)
    out = np.empty(llrs.shape)
    pos = llrs >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-llrs[pos]))
    e = np.exp(llrs[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def j_counts_from_traces(traces, gammas):
    """J(gamma) conditioning counts of sim._sim_block (sim.py:172-183):
    counts[k, gi, 0] = #(correct and D >= gamma), [..., 1] = #(wrong and D >= gamma),
    D = |p0(total) - p0(pre_total)| per VN at boundary k, correct = total >= 0."""
    traces = list(traces)
    n = traces[0].shape[1] // 2
    out = np.zeros((traces[0].shape[0], len(gammas), 2), np.int64)
    for tr in traces:
        for k in range(tr.shape[0]):
            tot, pre = tr[k, :n], tr[k, n:]
            d = np.abs(p0_vec(tot) - p0_vec(pre))
            correct = tot >= 0
            for gi, gm in enumerate(gammas):
                sel = d >= gm
                out[k, gi, 0] += int(np.sum(sel & correct))
                out[k, gi, 1] += int(np.sum(sel & ~correct))
    return out


def trace_golden_cases():
    z = np.load(GOLDEN / "trace.npz")
    return [(si, ast.literal_eval(str(s))) for si, s in enumerate(z["schedules"])]
