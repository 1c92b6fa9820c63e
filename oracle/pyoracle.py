"""ctypes binding of the C oracle (oracle/ldpc_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module.  The product path (paper_2102_11089_b200) never
does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
KINDS = {"flooding": 0, "rbp": 1, "cirbp": 2, "lmdrbp": 3, "slmdrbp": 4, "lmd_cirbp": 5,
         "me_cirbp": 6, "me_lmd_cirbp": 7, "layered": 8, "me_rbp": 9}
KERNELS = {"exact": 0, "minsum": 1}

_P = C.c_void_p
_I64 = C.c_int64
_LIBS = {}


def build(force=False):
    """Compile the oracle with its Makefile (gcc; no GPU needed)."""
    out = HERE / "build" / "libldpc_oracle.so"
    if force or not out.exists() or out.stat().st_mtime < (HERE / "ldpc_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    return out


def lib(single=False):
    key = "f32" if single else "f64"
    if key not in _LIBS:
        build()
        path = HERE / "build" / ("libldpc_oracle_f32.so" if single else "libldpc_oracle.so")
        L = C.CDLL(str(path))
        L.or_decode.restype = C.c_int
        L.or_decode.argtypes = ([_I64] * 3 + [_P] * 5 + [_P, C.c_int, C.c_int, C.c_int, _I64,
                                C.c_double, C.c_int, C.c_int, _I64] + [_P] * 9 + [_I64] + [_P] * 4)
        L.or_decode_batch.restype = C.c_int
        L.or_decode_batch.argtypes = ([_I64, C.c_int] + [_I64] * 3 + [_P] * 5 +
                                      [_P, C.c_int, C.c_int, C.c_int, _I64, C.c_double, C.c_int,
                                       C.c_int, _I64] + [_P] * 8)
        L.or_select_vns.restype = _I64
        L.or_select_vns.argtypes = [_P, _P, _I64, C.c_int, C.c_int, _I64, _P]
        L.or_set_dump_edges.restype = None
        L.or_set_dump_edges.argtypes = [_P, _P, _I64]
        L.or_set_rng_log.restype = None
        L.or_set_rng_log.argtypes = [_P, _I64]
        L.or_rng_log_len.restype = _I64
        L.or_set_dump.restype = None
        L.or_set_dump.argtypes = [_I64, _P, _P, _I64]
        L.or_rand_next.restype = _I64
        L.or_rand_next.argtypes = [_P]
        _LIBS[key] = L
    return _LIBS[key]


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _graph_arrays(g):
    return [np.ascontiguousarray(a, dtype=np.int64)
            for a in (g.edge_cn, g.edge_vn, g.cn_ptr, g.vn_ptr, g.vn_edges)]


def _seed64(seed):
    s = int(seed) & 0xFFFFFFFFFFFFFFFF
    return s - (1 << 64) if s >= (1 << 63) else s


def decode(g, chl, kind, kernel="exact", i_max=3, k_info=0, gamma=0.1, n_p=1, n_g=16, seed=0,
           want_trace=False, log_cap=0, single=False):
    """One frame through the oracle; returns a dict of numpy outputs."""
    L = lib(single)
    ga = _graph_arrays(g)
    N, M, E = g.n_vars, g.n_checks, g.n_edges
    chl = np.ascontiguousarray(chl, dtype=np.float64)
    out = {
        "u_hat": np.zeros(N, np.int8), "prop": np.zeros(1, np.int64), "converged": np.zeros(1, np.uint8),
        "counters": np.zeros(8, np.int64), "bit_errors_at": np.zeros(i_max + 1, np.int64),
        "info_bit_errors_at": np.zeros(i_max + 1, np.int64),
        "kappa_hits_iter": np.zeros(max(i_max, 1), np.int64),
        "kappa_trials_iter": np.zeros(max(i_max, 1), np.int64),
    }
    trace = np.zeros(((i_max + 1), 2 * N)) if want_trace else None
    le = np.zeros(max(log_cap, 1), np.int64)
    lc = np.zeros(max(log_cap, 1))
    lg = np.zeros(max(log_cap, 1))
    ll = np.zeros(1, np.int64)
    rc = L.or_decode(N, M, E, *[_p(a) for a in ga], _p(chl), KINDS[kind], KERNELS[kernel], i_max,
                     k_info, gamma, n_p, n_g, _seed64(seed), _p(out["u_hat"]), _p(out["prop"]),
                     _p(out["converged"]), _p(out["counters"]), _p(out["bit_errors_at"]),
                     _p(out["info_bit_errors_at"]), _p(out["kappa_hits_iter"]),
                     _p(out["kappa_trials_iter"]), _p(trace), log_cap, _p(le), _p(lc), _p(lg), _p(ll))
    if rc != 0:
        raise ValueError(f"oracle rejected kind {kind!r}")
    out["prop"] = int(out["prop"][0])
    out["converged"] = bool(out["converged"][0])
    if kind != "cirbp":
        out["kappa_hits_iter"] = np.zeros(0, np.int64)
        out["kappa_trials_iter"] = np.zeros(0, np.int64)
    else:
        out["kappa_hits_iter"] = out["kappa_hits_iter"][:i_max]
        out["kappa_trials_iter"] = out["kappa_trials_iter"][:i_max]
    if want_trace:
        out["trace_llrs"] = trace
    if log_cap:
        n = min(int(ll[0]), log_cap)
        out["log_edge"], out["log_c2v"], out["log_gap"] = le[:n], lc[:n], lg[:n]
        out["log_len"] = int(ll[0])
    return out


def decode_batch(g, chl, kind, kernel="exact", i_max=3, k_info=0, gamma=0.1, n_p=1, n_g=16,
                 seed=0, threads=None, single=False):
    """[B, N] frames on `threads` host threads (default: all cores)."""
    L = lib(single)
    ga = _graph_arrays(g)
    chl = np.ascontiguousarray(chl, dtype=np.float64)
    B, N = chl.shape
    I = i_max
    out = {
        "u_hat": np.zeros((B, N), np.int8), "prop": np.zeros(B, np.int64),
        "converged": np.zeros(B, np.uint8), "counters": np.zeros((B, 8), np.int64),
        "bit_errors_at": np.zeros((B, I + 1), np.int64),
        "info_bit_errors_at": np.zeros((B, I + 1), np.int64),
        "kappa_hits_iter": np.zeros((B, max(I, 1)), np.int64),
        "kappa_trials_iter": np.zeros((B, max(I, 1)), np.int64),
    }
    threads = threads or os.cpu_count() or 1
    L.or_decode_batch(B, threads, N, g.n_checks, g.n_edges, *[_p(a) for a in ga], _p(chl),
                      KINDS[kind], KERNELS[kernel], i_max, k_info, gamma, n_p, n_g, _seed64(seed),
                      _p(out["u_hat"]), _p(out["prop"]), _p(out["converged"]), _p(out["counters"]),
                      _p(out["bit_errors_at"]), _p(out["info_bit_errors_at"]),
                      _p(out["kappa_hits_iter"]), _p(out["kappa_trials_iter"]))
    out["converged"] = out["converged"].astype(bool)
    out["kappa_hits_iter"] = out["kappa_hits_iter"][:, :I]
    out["kappa_trials_iter"] = out["kappa_trials_iter"][:, :I]
    return out


def select_vns(ci, n_g, n_p, seed, mask=None):
    L = lib()
    ci = np.ascontiguousarray(ci, dtype=np.float64)
    mask = np.ones(len(ci), np.int8) if mask is None else np.ascontiguousarray(mask, np.int8)
    out = np.zeros(n_p, np.int64)
    cnt = L.or_select_vns(_p(ci), _p(mask), len(ci), n_g, n_p, _seed64(seed), _p(out))
    return out[:cnt]


def rand_next(state):
    st = np.array([_seed64(state)], np.int64)
    z = lib().or_rand_next(_p(st))
    return int(z), int(st[0])


def decode_dump(g, chl, step, **kw):
    """decode() with the oracle's ci / pre_total captured before update `step`."""
    L = lib(kw.get("single", False))
    ci = np.zeros(g.n_vars)
    pt = np.zeros(g.n_vars)
    rng = np.zeros(8192, np.int64)
    pre = np.zeros(g.n_edges)
    c2v = np.zeros(g.n_edges)
    L.or_set_dump_edges(_p(pre), _p(c2v), g.n_edges)
    L.or_set_dump(step, _p(ci), _p(pt), g.n_vars)
    L.or_set_rng_log(_p(rng), len(rng))
    try:
        kw.setdefault("log_cap", step + 2)
        r = decode(g, chl, **kw)
        nr = L.or_rng_log_len()
    finally:
        L.or_set_dump(-1, None, None, 0)
        L.or_set_dump_edges(None, None, 0)
        L.or_set_rng_log(None, 0)
    r["dump_ci"], r["dump_pretot"], r["rng_log"] = ci, pt, rng[:nr]
    r["dump_pre"], r["dump_c2v"] = pre, c2v
    return r
