"""Pin the CPU oracle against golden vectors produced by the reference itself.

Bit-exact: hard decisions, update counts, convergence, all 8 counters, bit
errors per boundary and kappa hits/trials, for every schedule and config in
tests/golden/*.npz (tests/golden/make_golden.py).
"""

import ast
import os

import numpy as np
import pytest

from oracle import pyoracle
from tests.util import golden_cases, load_code

pytestmark = pytest.mark.cpu


@pytest.mark.parametrize("fname,code_key,si,sched", golden_cases())
def test_oracle_matches_reference_golden(fname, code_key, si, sched):
    z = np.load(f"tests/golden/{fname}.npz")
    spec, g = load_code(code_key)
    llrs = z["llrs"].astype(np.float64)
    cfg = dict(kind="flooding", gamma=0.1, n_p=1, n_g=16, i_max=3, kernel="exact",
               selection_seed=0)
    cfg.update(sched)
    # BG1 cases at i_max 10 cost seconds per frame on the CPU: the oracle is
    # pinned on the first 8 of their 16 frames here (the GPU tests compare the
    # CUDA decoder with all 16 reference frames directly)
    nf = 8 if code_key == "C3" and cfg["i_max"] > 2 else len(llrs)
    llrs = llrs[:nf]
    out = pyoracle.decode_batch(g, llrs, cfg["kind"], cfg["kernel"], cfg["i_max"], spec.k_info,
                                cfg["gamma"], cfg["n_p"], cfg["n_g"], cfg["selection_seed"],
                                threads=os.cpu_count())
    t = f"s{si}"
    z = {k: z[k][:nf] for k in z.files if k.startswith(t + "_")}
    np.testing.assert_array_equal(np.packbits(out["u_hat"], axis=1), z[f"{t}_u_hat"])
    np.testing.assert_array_equal(out["prop"], z[f"{t}_prop"])
    np.testing.assert_array_equal(out["converged"], z[f"{t}_converged"])
    np.testing.assert_array_equal(out["counters"], z[f"{t}_counters"])
    np.testing.assert_array_equal(out["bit_errors_at"], z[f"{t}_biterr"])
    np.testing.assert_array_equal(out["info_bit_errors_at"], z[f"{t}_biterr_info"])
    if cfg["kind"] == "cirbp":
        np.testing.assert_array_equal(out["kappa_hits_iter"], z[f"{t}_kh"])
        np.testing.assert_array_equal(out["kappa_trials_iter"], z[f"{t}_kt"])


def test_oracle_single_frame_api_matches_batch():
    spec, g = load_code("C0")
    z = np.load("tests/golden/c0.npz")
    llr = z["llrs"][3].astype(np.float64)
    one = pyoracle.decode(g, llr, "cirbp", i_max=5, k_info=spec.k_info)
    many = pyoracle.decode_batch(g, llr[None], "cirbp", i_max=5, k_info=spec.k_info, threads=1)
    assert one["prop"] == many["prop"][0]
    np.testing.assert_array_equal(one["counters"], many["counters"][0])


def test_kats():
    k = np.load("tests/golden/kat.npz")
    for (n_g, n_p, seed) in ((16, 4, 0), (16, 64, 3), (4, 100, 99), (1, 10, 5), (64, 7, 2**63 + 11)):
        got = pyoracle.select_vns(k["select_ci"], n_g, n_p, seed)
        np.testing.assert_array_equal(got, k[f"select_{n_g}_{n_p}_{seed}"])
    np.testing.assert_array_equal(pyoracle.select_vns([0.9, 0.7, 0.3, 0.1], 4, 2, 0), [0, 1])
    seq = []
    for seed in (0, 1, 12345, -1, 2**62):
        st, row = seed, []
        for _ in range(8):
            z, st = pyoracle.rand_next(st)
            row.append(z)
        seq.append(row)
    np.testing.assert_array_equal(np.array(seq, np.int64), k["rand_seq"])
    assert abs(float(k["c2v_22"]) - 1.3250027) < 1e-6
    assert float(k["c2v_minsum"]) == -2.0
    assert float(k["c2v_zero"]) == 0.0
    np.testing.assert_array_equal(k["select_vns_spec"], [0, 1])


def test_me_rbp_np1_equals_rbp():
    """Definition check for the new ME-RBP schedule: n_p = 1 reproduces RBP."""
    spec, g = load_code("C0")
    llrs = np.load("tests/golden/c0.npz")["llrs"][:12].astype(np.float64)
    a = pyoracle.decode_batch(g, llrs, "rbp", i_max=5, k_info=spec.k_info)
    b = pyoracle.decode_batch(g, llrs, "me_rbp", i_max=5, k_info=spec.k_info, n_p=1)
    for key in ("u_hat", "prop", "converged", "counters", "bit_errors_at"):
        np.testing.assert_array_equal(a[key], b[key])


def test_layered_counts_and_convergence():
    spec, g = load_code("C0")
    llrs = np.load("tests/golden/c0.npz")["llrs"][:20].astype(np.float64)
    lay = pyoracle.decode_batch(g, llrs, "layered", i_max=5, k_info=spec.k_info)
    fl = pyoracle.decode_batch(g, llrs, "flooding", i_max=5, k_info=spec.k_info)
    assert (lay["prop"] % g.n_edges == 0).all()
    assert (lay["counters"][:, 0] == lay["prop"]).all()
    # layered converges at least as often as flooding on the same frames
    assert lay["converged"].sum() >= fl["converged"].sum()


def test_golden_schedule_lists_parse():
    for fname, _, _, sched in golden_cases():
        assert isinstance(sched, dict)
    z = np.load("tests/golden/c0.npz")
    assert all(isinstance(ast.literal_eval(s), dict) for s in z["schedules"])


@pytest.mark.parametrize("si,sched", __import__("tests.util", fromlist=["x"]).trace_golden_cases())
def test_oracle_trace_matches_reference(si, sched):
    """want_trace rows (totals, pre-totals per boundary; E:192-217, E:768-782)."""
    import hashlib
    z = np.load("tests/golden/trace.npz")
    spec, g = load_code("C0")
    cfg = dict(kind="flooding", gamma=0.1, n_p=1, n_g=16, i_max=3, kernel="exact", selection_seed=0)
    cfg.update(sched)
    for f, row in enumerate(z["llrs"].astype(np.float64)):
        r = pyoracle.decode(g, row, cfg["kind"], cfg["kernel"], cfg["i_max"], spec.k_info, cfg["gamma"],
                            cfg["n_p"], cfg["n_g"], cfg["selection_seed"], want_trace=True)
        tr = np.ascontiguousarray(r["trace_llrs"], np.float64)
        if f == 0:
            np.testing.assert_array_equal(tr, z[f"s{si}_trace0"])
        assert hashlib.sha256(tr.tobytes()).hexdigest() == z[f"s{si}_sha"][f], (sched, f)


def test_oracle_j_gamma_counts_match_reference():
    """mc_j_gamma (sim.py:339-353) counts from oracle traces of the same frames."""
    from paper_2102_11089_b200.channel import llr_batch
    from tests.util import j_counts_from_traces
    z = np.load("tests/golden/trace.npz")
    spec, g = load_code("C0")
    gam = list(z["j_gammas"])
    llrs = llr_batch(spec, float(z["j_ebn0"]), int(z["j_seed"]), 0, int(z["j_frames"]), dtype=np.float64)
    for ci, case in enumerate(z["j_cases"]):
        cfg = dict(kind="flooding", gamma=0.1, n_p=1, n_g=16, i_max=3, kernel="exact", selection_seed=0)
        cfg.update(ast.literal_eval(str(case)))
        traces = [pyoracle.decode(g, row, cfg["kind"], cfg["kernel"], cfg["i_max"], spec.k_info,
                                  cfg["gamma"], cfg["n_p"], cfg["n_g"], cfg["selection_seed"],
                                  want_trace=True)["trace_llrs"] for row in llrs]
        np.testing.assert_array_equal(j_counts_from_traces(traces, gam), z["j_counts"][ci], err_msg=str(case))


def test_oracle_rbp_equals_reference_stepwise_decoder():
    """The reference's stepwise DecoderState (kernels.py:98-181) driven by the
    first residual maximum is RBP (E:355-385): the oracle's RBP step log (edge,
    committed C2V) reproduces tests/golden/steps.npz update for update."""
    z = np.load("tests/golden/steps.npz")
    for i in range(int(z["n_cases"])):
        case = ast.literal_eval(str(z[f"c{i}_case"]))
        spec, g = load_code(case["code"])
        for f, llr in enumerate(z[f"c{i}_llrs"]):
            r = pyoracle.decode(g, llr.astype(np.float64), "rbp", case["kernel"], 1, spec.k_info, log_cap=1000)
            np.testing.assert_array_equal(r["log_edge"][:1000], z[f"c{i}_edges"][f], err_msg=str((case, f)))
            np.testing.assert_array_equal(r["log_c2v"][:1000], z[f"c{i}_c2v"][f], err_msg=str((case, f)))
