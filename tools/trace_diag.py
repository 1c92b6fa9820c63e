import sys; sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch, ast
from oracle import pyoracle
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch, results_to_numpy
from paper_2102_11089_b200.channel import llr_batch
from tests.util import load_code
for key in ("C0", "C1"):
    spec, g = load_code(key)
    llrs = llr_batch(spec, 2.0, seed=5, start=0, count=100)
    for kind in ["flooding", "layered", "rbp", "cirbp", "lmdrbp", "me_cirbp", "me_rbp"]:
        cfg = ScheduleConfig(kind=kind, i_max=3, n_p=4)
        got = results_to_numpy(decode_batch(spec, torch.from_numpy(llrs).cuda(), cfg, want_trace=True), kind, 3)
        mx = 0; mrel = 0; nsame = 0; nbit = 0
        for f in range(len(llrs)):
            r = pyoracle.decode(g, llrs[f].astype(np.float64), kind, "exact", 3, spec.k_info, 0.1, 4, 16, 0, want_trace=True)
            if not ((got["u_hat"][f] == r["u_hat"]).all() and got["prop"][f] == r["prop"]):
                continue
            nsame += 1
            a, b = got["trace_llrs"][f], r["trace_llrs"]
            d = np.abs(a - b)
            mx = max(mx, d.max()); mrel = max(mrel, (d / np.maximum(np.abs(b), 1e-300)).max())
            nbit += (d == 0).all()
        print(key, kind, "same", nsame, "bitexact", nbit, "maxabs %.3g maxrel %.3g" % (mx, mrel), flush=True)
