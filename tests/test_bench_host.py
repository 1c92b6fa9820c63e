"""bench.py host logic (no GPU): algorithmic bytes per update
and the FER-vs-oracle Clopper-Pearson interval."""

import numpy as np
from scipy.stats import binomtest

import bench


def test_clopper_pearson_matches_scipy_exact():
    for k, n in [(0, 50), (5, 100), (668, 8464), (8464, 8464), (1, 1)]:
        lo, hi = bench.clopper_pearson(k, n)
        ci = binomtest(k, n).proportion_ci(confidence_level=0.95, method="exact")
        assert abs(lo - ci.low) < 1e-9 and abs(hi - ci.high) < 1e-9


def test_bytes_per_update_formulas():
    # flooding / layered: 16 + 8N/E and 16 B (fp32 units), doubled for fp64
    c = np.zeros((4, 8), np.int64)
    c[:, 0] = 100
    assert bench.bytes_per_update("flooding", c, E=1512, N=504, elem=4) == 16 + 8 * 504 / 1512
    assert bench.bytes_per_update("layered", c, E=1512, N=504, elem=8) == 32
    # dynamic: 20 (+8 CI) + (12V + 28R + 8I)/P; C0 RBP numbers from SURVEY (V/P=2, R/P=10) -> 324 B
    c[:, 1] = 200
    c[:, 2] = 1000
    assert abs(bench.bytes_per_update("rbp", c, E=1512, N=504, elem=4) - 324.0) < 1e-9
    c[:, 3] = 1000
    assert abs(bench.bytes_per_update("cirbp", c, E=1512, N=504, elem=4) - 412.0) < 1e-9
