"""ctypes binding of the CUDA C-ABI library (include/ldpc_b200.h).

The product decode path goes through here and nowhere else: if the built
library is missing the import fails loudly -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("LDPC_B200_LIB", PKG / "lib" / "libldpc_b200.so"))

LDPC_OK = 0
ERRORS = {-1: "invalid argument", -2: "unsupported", -3: "CUDA error", -4: "workspace too small"}


class LdpcSched(C.Structure):
    _fields_ = [("kind", C.c_int32), ("kernel", C.c_int32), ("i_max", C.c_int32),
                ("n_p", C.c_int32), ("n_g", C.c_int32), ("k_info", C.c_int32),
                ("gamma", C.c_double), ("selection_seed", C.c_int64),
                ("precision", C.c_int32), ("llr_f64", C.c_int32),
                ("max_resident", C.c_int32), ("placement", C.c_int32),
                ("want_trace", C.c_int32), ("variant", C.c_int32)]


# ldpc_sched_t.variant bits (include/ldpc_b200.h)
VARIANTS = {"fixed_phase": 0x1, "fixed_tile": 0x2, "fixed_pipe": 0x3, "check_tma": 0x4,
            "check_legacy": 0x8, "no_layered_sign": 0x10, "lanes32": 0x20, "lanes16": 0x40,
            "full_tree": 0x80, "me_pairs": 0x100}


def variant_bits(names):
    bits = 0
    for n in (names.split(",") if isinstance(names, str) else names or ()):
        if n:
            bits |= VARIANTS[n]
    return bits


# every exported symbol of include/ldpc_b200.h
EXPORTS = ("ldpc_graph_create", "ldpc_graph_destroy", "ldpc_graph_info", "ldpc_workspace_size",
           "ldpc_decode", "ldpc_decode_traced", "ldpc_select_vns", "ldpc_set_step_log", "ldpc_set_state_dump",
           "ldpc_generate_awgn", "ldpc_replay_workspace_size", "ldpc_decode_replay",
           "ldpc_last_launch_count",
           "ldpc_strerror", "ldpc_version")

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryMissing(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the decoder has no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    P, I32, I64, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
    L.ldpc_graph_create.argtypes = [P, P, P, P, P, I32, I32, I32, C.POINTER(P)]
    L.ldpc_graph_destroy.argtypes = [P]
    L.ldpc_graph_info.argtypes = [P, P]
    L.ldpc_workspace_size.argtypes = [P, C.POINTER(LdpcSched), I64, C.POINTER(SZ)]
    L.ldpc_decode.argtypes = [P, P, I64, C.POINTER(LdpcSched)] + [P] * 8 + [P, SZ, P]
    L.ldpc_decode_traced.argtypes = [P, P, I64, C.POINTER(LdpcSched)] + [P] * 8 + [P, P, I32, P] + [P, SZ, P]
    L.ldpc_select_vns.argtypes = [P, P, I32, I32, I32, I64, P, P, P]
    L.ldpc_set_step_log.argtypes = [P, I32]
    L.ldpc_generate_awgn.argtypes = [I32, I32, I64, C.c_double, C.c_uint64, I64, P, I32, P]
    L.ldpc_set_state_dump.argtypes = [I64, P]
    L.ldpc_replay_workspace_size.argtypes = [P, C.POINTER(LdpcSched), I64, C.POINTER(SZ)]
    L.ldpc_decode_replay.argtypes = [P, P, I64, C.POINTER(LdpcSched), P, I32, P, P, P, P, SZ, P]
    L.ldpc_last_launch_count.argtypes = []
    L.ldpc_strerror.argtypes = [C.c_int]
    L.ldpc_strerror.restype = C.c_char_p
    L.ldpc_version.argtypes = []
    for name in EXPORTS:
        if name not in ("ldpc_strerror",):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(rc, what):
    if rc != LDPC_OK:
        msg = lib().ldpc_strerror(rc).decode()
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: {msg} (code {rc})")
