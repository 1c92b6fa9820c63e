"""Shared test helpers (no GPU, no reference import)."""

import ast
import functools
from pathlib import Path

import numpy as np

from paper_2102_11089_b200 import configs
from paper_2102_11089_b200.codes import build_tanner

GOLDEN = Path(__file__).resolve().parent / "golden"
FILES = {"c0": "C0", "c1": "C1", "c2": "C2", "c3": "C3"}


@functools.lru_cache(maxsize=None)
def load_code(key):
    spec = {"C0": configs.make_c0_code, "C1": configs.make_c1_code, "C2": configs.make_c2_code,
            "C3": configs.make_c3_code}[key]()
    return spec, build_tanner(spec.h)


def golden_cases(files=("c0", "c1", "c2", "c3")):
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
