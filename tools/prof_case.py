"""One decode launch of a chosen case (for ncu / timing).

    python tools/prof_case.py CODE KIND NFRAMES [global] [f32] [n_p=4]
A 1-frame warm-up launch precedes the measured launch (ncu: -s 1 -c 1).
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2102_11089_b200 import configs  # noqa: E402
from paper_2102_11089_b200.channel import llr_batch  # noqa: E402
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch  # noqa: E402

key, kind, nfr = sys.argv[1], sys.argv[2], int(sys.argv[3])
flags = sys.argv[4:]
placement = next((f for f in flags if f in ("smem", "split", "hbm", "trees")), "hbm" if "global" in flags else "auto")
prec = "f32" if "f32" in flags else "f64"
n_p = 4
imax_over = None
max_res = 0
for f in flags:
    if f.startswith("res="):
        max_res = int(f[4:])
    if f.startswith("n_p="):
        n_p = int(f[4:])
    if f.startswith("imax="):
        imax_over = int(f[5:])
spec = getattr(configs, f"make_{('c2' if key == 'C4' else key).lower()}_code")()
imax = {"C0": 5, "C1": 3, "C2": 3, "C3": 10, "C4": 20}[key]
eb = {"C0": 2.0, "C1": 2.0, "C2": 1.0, "C3": 1.0, "C4": 0.0}[key]
if key == "C4":
    spec = configs.make_c2_code()
llr = torch.from_numpy(llr_batch(spec, eb, 0, 0, nfr)).cuda()
imax = imax_over or imax
cfg = ScheduleConfig(kind=kind, i_max=imax, n_p=n_p, precision=prec)
decode_batch(spec, llr[:1], cfg, placement=placement, max_resident=max_res)
torch.cuda.synchronize()
reps = int(next((f[5:] for f in flags if f.startswith("reps=")), "1"))
dts = []
for _ in range(reps):  # ncu: -s 1 -c 1 captures the first of these
    t = time.time()
    out = decode_batch(spec, llr, cfg, placement=placement, max_resident=max_res)
    torch.cuda.synchronize()
    dts.append(time.time() - t)
dt = min(dts)
upd = int(out["counters"][:, 0].sum())
print(f"{key} {kind} {prec} {placement} res={max_res} frames={nfr} time={dt*1e3:.2f} ms updates={upd} "
      f"upd/s={upd/dt:.3e} frames/s={nfr/dt:.3e} us/update/warp-est={dt*1e6/max(1,upd/nfr):.2f}")
