"""Quick GPU parity probe: every schedule on small batches vs the CPU oracle."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import pyoracle  # noqa: E402
from paper_2102_11089_b200.channel import llr_batch  # noqa: E402
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch, results_to_numpy  # noqa: E402
from tests.util import load_code  # noqa: E402

codes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C0"]
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else [
    "flooding", "layered", "rbp", "cirbp", "lmdrbp", "slmdrbp", "lmd_cirbp", "me_cirbp",
    "me_lmd_cirbp", "me_rbp"]
nfr = int(sys.argv[3]) if len(sys.argv) > 3 else 256
for key in codes:
    spec, g = load_code(key)
    imax = {"C0": 5, "C1": 3, "C2": 3, "C3": 2}[key]
    eb = {"C0": 2.0, "C1": 2.0, "C2": 1.0, "C3": 1.0}[key]
    llr = llr_batch(spec, eb, 0, 0, nfr)
    for kind in kinds:
        for fg in ("auto", "smem", "split", "trees", "hbm"):
            cfg = ScheduleConfig(kind=kind, i_max=imax, n_p=4)
            t = time.time()
            try:
                out = decode_batch(spec, torch.from_numpy(llr).cuda(), cfg, placement=fg)
            except RuntimeError as ex:
                print(key, kind, fg, 'skipped:', ex); continue
            torch.cuda.synchronize()
            dt = time.time() - t
            got = results_to_numpy(out, kind, imax)
            ref = pyoracle.decode_batch(g, llr.astype(np.float64), kind, i_max=imax, k_info=spec.k_info, n_p=4)
            same = (got["u_hat"] == ref["u_hat"]).all(1) & (got["prop"] == ref["prop"])
            cnt = (got["counters"] == ref["counters"]).all(1)
            be = (got["bit_errors_at"] == ref["bit_errors_at"]).all(1)
            print(f"{key} {kind:13s} {fg:5s} same={same.mean():.4f} counters={cnt.mean():.4f} "
                  f"biterr={be.mean():.4f} conv={np.mean(got['converged'] == ref['converged']):.4f} "
                  f"gpu {dt*1e3:.1f} ms", flush=True)
            if not same.all():
                b = int(np.flatnonzero(~same)[0])
                print("   first bad frame", b, "prop gpu/ref", got["prop"][b], ref["prop"][b],
                      "counters gpu", got["counters"][b].tolist(), "ref", ref["counters"][b].tolist())
