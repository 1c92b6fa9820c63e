"""Host-side logic of the GPU Monte Carlo harness (paper_2102_11089_b200/sim.py):
validation, per-block tallies and record formatting, checked on CPU tensors
against the reference harness's rules (sim.py:47-56, 145-171, 269-300)."""

import numpy as np
import pytest
import torch

from paper_2102_11089_b200 import sim
from paper_2102_11089_b200.schedules import ScheduleConfig
from tests.util import load_code

pytestmark = pytest.mark.cpu


def test_campaign_validation_messages():
    s = [ScheduleConfig(kind="rbp")]
    with pytest.raises(ValueError, match="min_frame_errors must be >= 1"):
        sim.Campaign(code="C0", schedules=s, snr_grid=[1.0], min_frame_errors=0)
    with pytest.raises(ValueError, match="max_frames must be >= 1"):
        sim.Campaign(code="C0", schedules=s, snr_grid=[1.0], max_frames=0)
    with pytest.raises(ValueError, match="snr grid must be non-empty"):
        sim.Campaign(code="C0", schedules=s, snr_grid=[])
    with pytest.raises(ValueError, match="at least one schedule is required"):
        sim.Campaign(code="C0", schedules=[], snr_grid=[1.0])


def _fake_out(B, I, rng):
    be = rng.integers(0, 3, size=(B, I + 1)).astype(np.int32)
    return {
        "bit_errors_at": torch.from_numpy(be),
        "info_bit_errors_at": torch.from_numpy((be // 2).astype(np.int32)),
        "converged": torch.from_numpy((be[:, I] == 0).astype(np.uint8)),
        "counters": torch.from_numpy(rng.integers(0, 100, size=(B, 8))),
        "kappa_hits_iter": torch.from_numpy(rng.integers(0, 5, size=(B, max(I, 1))).astype(np.int32)),
        "kappa_trials_iter": torch.from_numpy(rng.integers(5, 9, size=(B, max(I, 1))).astype(np.int32)),
    }


def test_block_tallies_follow_reference_rules():
    rng = np.random.default_rng(0)
    I, B = 3, 700
    out = _fake_out(B, I, rng)
    t = sim._block_tallies(out, I, 3, B).numpy()
    be = out["bit_errors_at"].numpy()
    for b in range(3):
        sl = slice(b * 256, min(B, (b + 1) * 256))
        assert t[b, 0] == int((be[sl, I] > 0).sum())                     # SIM:152-154
        assert t[b, 1] == int(out["info_bit_errors_at"].numpy()[sl, I].sum())
        assert t[b, 2] == int(out["converged"].numpy()[sl].sum())
        np.testing.assert_array_equal(t[b, 3:11], out["counters"].numpy()[sl].sum(0))
        np.testing.assert_array_equal(t[b, 11:11 + I + 1], (be[sl] > 0).sum(0))  # SIM:165
        assert t[b, -1] == sl.stop - sl.start


def test_record_fields_and_csv():
    spec, g = load_code("C0")
    cfg = ScheduleConfig(kind="cirbp", i_max=2)
    acc = {"frames": 512, "frame_errors": 7, "bit_errors": 30, "converged": 505,
           "counters": np.array([1000, 2000, 3000, 3000, 50, 0, 3, 10]),
           "frame_errors_at": np.array([400, 20, 7]), "bit_errors_at": np.array([900, 60, 30]),
           "kappa_hits_iter": np.array([2, 1]), "kappa_trials_iter": np.array([6, 0])}
    r = sim._record_from_cell(spec, cfg, 1.5, 0, acc, 0.1)
    assert r.fer == 7 / 512 and r.ber == 30 / (512 * spec.k_info)
    assert r.kappa == 0.3 and r.kappa_per_iteration == [2 / 6, None]
    assert r.mean_iterations == 1000 / (512 * g.n_edges)
    text = sim.records_to_csv([r])
    head, row = text.strip().split("\n")
    assert head.split(",") == list(sim.SimRecord.CSV_COLUMNS)
    assert row.split(",")[:3] == [spec.label, "cirbp", "0.1"]
    assert sim.records_to_jsonl([r]).count("\n") == 1
