"""Per-update parity with the reference's stepwise decoder (kernels.py:98-181).

tests/golden/steps.npz holds, for C0-C2 frames, the first 1000 updates of the
reference's own DecoderState.propagate (edge chosen as the first residual
maximum), the C2V value each update committed, the state after them and the
reference's recompute_all audit of that state (make_golden.py --only-steps).
The GPU replays the same edge sequence (ldpc_decode_replay):
* float64: every committed value and the final c2v / pre_c2v / total /
  pre_total / ci within 1e-12 relative of the reference (CUDA's float64
  tanh / atanh / exp and glibc's differ in the last ulp on some arguments, so
  message values agree to a few ulps; decisions, update counts and counters of
  whole decodes are compared exactly in test_gpu_parity.py) and the counters
  identical;
* the audit: the GPU's incrementally maintained state equals a from-scratch
  recompute (the reference's recompute_all arrays) to float64 rounding;
* float32 (phi-domain check nodes): every committed value within 1e-4
  relative (absolute below 1), saturated messages included -- the replay
  follows the reference's sequence, so no near-tie can end the comparison.
"""

import ast

import numpy as np
import pytest
import torch

from paper_2102_11089_b200.schedules import decode_replay
from tests.util import GOLDEN, load_code

pytestmark = pytest.mark.gpu

Z = np.load(GOLDEN / "steps.npz")
CASES = [(i, ast.literal_eval(str(Z[f"c{i}_case"]))) for i in range(int(Z["n_cases"]))]


def _replay(i, case, precision="f64"):
    spec, g = load_code(case["code"])
    out = decode_replay(spec, Z[f"c{i}_llrs"], Z[f"c{i}_edges"], kernel=case["kernel"], precision=precision)
    torch.cuda.synchronize()
    return spec, g, {k: v.cpu().numpy() for k, v in out.items() if not k.startswith("_")}


@pytest.mark.parametrize("i,case", CASES)
def test_replay_f64_matches_reference_stepwise(i, case):
    spec, g, r = _replay(i, case)
    np.testing.assert_allclose(r["c2v_trace"], Z[f"c{i}_c2v"], rtol=1e-12, atol=1e-13)
    for k_gpu, k_ref in (("c2v", "s_c2v"), ("pre_c2v", "s_pre"), ("total", "s_total"), ("pre_total", "s_pretot")):
        np.testing.assert_allclose(r[k_gpu], Z[f"c{i}_{k_ref}"], rtol=1e-12, atol=1e-12, err_msg=k_gpu)
    np.testing.assert_allclose(r["ci"], Z[f"c{i}_s_ci"], rtol=1e-9, atol=1e-13)
    np.testing.assert_array_equal(r["counters"][:, :4], Z[f"c{i}_counters"][:, :4])


@pytest.mark.parametrize("i,case", CASES)
def test_replay_state_passes_recompute_audit(i, case):
    """recompute_all (kernels.py:161-181): totals, pre-totals and CI rebuilt
    from the message arrays agree with the GPU's incrementally maintained
    ones.  (Residuals are not audited: the reference's incremental pre_c2v of
    the other edges of m* is deliberately not refreshed (E:143-144, E:156-157),
    so |pre - c2v| of the incremental state differs from recompute_all's
    residual in the reference itself; the GPU reproduces the incremental
    one, compared in the test above.)"""
    from tests.util import p0_vec
    spec, g, r = _replay(i, case)
    # totals from the C2V messages: the reference's own recompute
    np.testing.assert_allclose(r["total"], Z[f"c{i}_a_total"], rtol=1e-9, atol=1e-9)
    # pre-totals and CI from the GPU's own pre_c2v / totals (recompute_all's
    # formulas, K:175-180): the incremental upkeep is consistent
    chl = Z[f"c{i}_llrs"].astype(np.float64)
    for f in range(len(chl)):
        pt = chl[f].copy()
        np.add.at(pt, g.edge_vn, r["pre_c2v"][f])
        np.testing.assert_allclose(r["pre_total"][f], pt, rtol=1e-9, atol=1e-9)
        ci = np.abs(p0_vec(r["total"][f]) - p0_vec(r["pre_total"][f]))
        np.testing.assert_allclose(r["ci"][f], ci, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("i,case", CASES)
def test_replay_f32_within_1e4_of_reference(i, case):
    spec, g, r = _replay(i, case, precision="f32")
    x, y = Z[f"c{i}_c2v"], r["c2v_trace"]
    np.testing.assert_array_less(np.abs(x - y), 1e-4 * np.maximum(np.abs(x), 1.0) + 1e-12)
    if case["ebn0"] >= 6.0:
        assert (np.abs(x) > 28.0).any()  # saturated messages were compared


def test_replay_rejects_bad_edges():
    spec, g = load_code("C0")
    llr = np.zeros((1, g.n_vars), np.float32)
    with pytest.raises(ValueError):
        decode_replay(spec, llr, np.array([[g.n_edges]]))
    with pytest.raises(ValueError):
        decode_replay(spec, llr, np.zeros((2, 3), np.int32))
