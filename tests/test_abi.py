"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/ldpc_b200.h declares, and the Python API mirrors the reference's
names and validation (no GPU needed)."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.cpu

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "ldpc_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ldpc_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported():
    from paper_2102_11089_b200 import _native
    L = _native.lib()
    names = _declared()
    assert len(names) >= 9
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_native.EXPORTS)
    assert L.ldpc_version() >= 10000
    assert L.ldpc_strerror(-1).decode() == "invalid argument"


def test_abi_rejects_bad_graphs_without_gpu():
    from paper_2102_11089_b200 import _native
    L = _native.lib()
    h = C.c_void_p()
    z = np.zeros(4, np.int32)
    p = z.ctypes.data_as(C.c_void_p)
    assert L.ldpc_graph_create(p, p, p, p, p, 0, 1, 1, C.byref(h)) == -1
    # unsorted edges are rejected before any device allocation
    ecn = np.array([1, 0], np.int32)
    evn = np.array([0, 0], np.int32)
    cptr = np.array([0, 1, 2], np.int32)
    vptr = np.array([0, 2], np.int32)
    ved = np.array([0, 1], np.int32)
    args = [a.ctypes.data_as(C.c_void_p) for a in (ecn, evn, cptr, vptr, ved)]
    assert L.ldpc_graph_create(*args, 1, 2, 2, C.byref(h)) == -1


def test_schedule_config_validation_matches_reference():
    from paper_2102_11089_b200.schedules import ScheduleConfig
    with pytest.raises(ValueError, match="unknown schedule kind"):
        ScheduleConfig(kind="nope")
    with pytest.raises(ValueError, match=r"gamma must lie in \[0, 1\)"):
        ScheduleConfig(kind="cirbp", gamma=1.0)
    with pytest.raises(ValueError, match="n_p and n_g must be >= 1"):
        ScheduleConfig(kind="me_cirbp", n_p=0)
    with pytest.raises(ValueError, match="i_max must be >= 0"):
        ScheduleConfig(kind="rbp", i_max=-1)
    with pytest.raises(ValueError, match="unknown kernel"):
        ScheduleConfig(kind="rbp", kernel="fast")
    cfg = ScheduleConfig(kind="rbp")
    assert (cfg.gamma, cfg.n_p, cfg.n_g, cfg.i_max, cfg.kernel, cfg.selection_seed) == \
        (0.1, 1, 16, 3, "exact", 0)  # schedules.py:26-32


def test_api_names_mirror_reference():
    import paper_2102_11089_b200 as P
    from paper_2102_11089_b200 import schedules
    for name in ("decode", "select_vns", "ScheduleConfig", "DecodeResult", "build_tanner",
                 "make_random_regular_code", "generate_frame", "ebn0_to_sigma", "Counters"):
        assert hasattr(P, name)
    for k in ("flooding", "rbp", "cirbp", "lmdrbp", "lmd_cirbp", "me_cirbp", "me_lmd_cirbp"):
        assert hasattr(schedules, f"decode_{k}")
