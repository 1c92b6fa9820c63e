"""GPU checks of the boundary itself (stream ordering, select_vns KATs,
engine pins through ldpc_sched_t.variant)."""

import numpy as np
import pytest
import torch

from paper_2102_11089_b200.channel import llr_batch
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch, results_to_numpy, select_vns
from tests.util import GOLDEN, load_code

pytestmark = pytest.mark.gpu


def test_select_vns_gpu_matches_reference_kats():
    """ldpc_select_vns (the GPU _select_vns, E:293-352) against the reference's
    own select_vns outputs (tests/golden/kat.npz, schedules.py:60-79)."""
    k = np.load(GOLDEN / "kat.npz")
    for (n_g, n_p, seed) in ((16, 4, 0), (16, 64, 3), (4, 100, 99), (1, 10, 5), (64, 7, 2**63 + 11)):
        got, _ = select_vns(k["select_ci"], n_g, n_p, seed)
        np.testing.assert_array_equal(got, k[f"select_{n_g}_{n_p}_{seed}"], err_msg=str((n_g, n_p, seed)))
    got, _ = select_vns([0.9, 0.7, 0.3, 0.1], 4, 2, 0)
    np.testing.assert_array_equal(got, k["select_vns_spec"])
    with pytest.raises(ValueError):
        select_vns([0.5, 0.2], 4, 3, 0)


@pytest.mark.parametrize("kind", ["cirbp", "me_cirbp", "layered"])
def test_two_streams_concurrently(kind):
    """Two decodes of different batches queued on two streams at once give the
    same answers as one after the other: each stream has its own workspace
    (DeviceGraph.workspace), allocated on that stream."""
    spec, g = load_code("C1")
    cfg = ScheduleConfig(kind=kind, i_max=3, n_p=4)
    a_in = torch.from_numpy(llr_batch(spec, 2.0, seed=0, start=0, count=3000)).cuda()
    b_in = torch.from_numpy(llr_batch(spec, 1.5, seed=1, start=0, count=2000)).cuda()
    ref_a = results_to_numpy(decode_batch(spec, a_in, cfg), kind, 3)
    ref_b = results_to_numpy(decode_batch(spec, b_in, cfg), kind, 3)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    outs = []
    for _ in range(2):
        oa = decode_batch(spec, a_in, cfg, stream=s1)
        ob = decode_batch(spec, b_in, cfg, stream=s2)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        ga, gb = results_to_numpy(oa, kind, 3), results_to_numpy(ob, kind, 3)
        for key in ("u_hat", "prop", "counters", "bit_errors_at"):
            np.testing.assert_array_equal(ga[key], ref_a[key], err_msg=key)
            np.testing.assert_array_equal(gb[key], ref_b[key], err_msg=key)


def test_variant_bits_validated():
    from paper_2102_11089_b200 import _native
    spec, g = load_code("C0")
    llrs = torch.zeros((2, g.n_vars), device="cuda")
    with pytest.raises(ValueError):
        decode_batch(spec, llrs, ScheduleConfig(kind="rbp"), variant=0x1000)
    with pytest.raises(ValueError):
        decode_batch(spec, llrs, ScheduleConfig(kind="rbp"), variant="lanes32,lanes16")
    assert _native.variant_bits("fixed_tile,check_tma") == 0x6


@pytest.mark.parametrize("code_key,eb,i_max,count,n_p", [("C0", 1.5, 4, 600, 4), ("C1", 2.0, 3, 800, 4),
                                                          ("C2", 1.0, 3, 300, 16), ("C3", 1.0, 2, 24, 64)])
@pytest.mark.parametrize("kind", ["me_cirbp", "me_lmd_cirbp"])
def test_me_round_pairing_is_exact(code_key, eb, i_max, count, n_p, kind):
    """Multi-edge rounds with disjoint consecutive VN pairs applied on the two
    half-warps (ldpc_sched_t.variant ME_PAIRS) == strictly one VN at a time:
    every output bit-identical (the reference's sequential order, E:625-632)."""
    spec, g = load_code(code_key)
    llrs = torch.from_numpy(llr_batch(spec, eb, seed=8, start=0, count=count)).cuda()
    cfg = ScheduleConfig(kind=kind, i_max=i_max, n_p=n_p)
    a = results_to_numpy(decode_batch(spec, llrs, cfg, variant="me_pairs"), kind, i_max)
    b = results_to_numpy(decode_batch(spec, llrs, cfg), kind, i_max)
    for key in ("u_hat", "prop", "converged", "counters", "bit_errors_at", "info_bit_errors_at"):
        np.testing.assert_array_equal(a[key], b[key], err_msg=key)
