"""Compare the GPU's update sequence with the oracle's for chosen golden frames."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import pyoracle
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch_logged
from tests.util import load_code
fname, key, kind, frames = sys.argv[1], sys.argv[2], sys.argv[3], [int(x) for x in sys.argv[4].split(",")]
placement = sys.argv[5] if len(sys.argv) > 5 else "auto"
kernel = sys.argv[6] if len(sys.argv) > 6 else "exact"
z = np.load(f"tests/golden/{fname}.npz")
spec, g = load_code(key)
imax = 5 if key == "C0" else 3
llr = z["llrs"][frames]
cfg = ScheduleConfig(kind=kind, i_max=imax, n_p=4, kernel=kernel)
out = decode_batch_logged(spec, torch.from_numpy(llr).cuda(), cfg, log_cap=8000, placement=placement)
glog = out["step_log"].cpu().numpy()
gval = out["step_c2v"].cpu().numpy()
for i, f in enumerate(frames):
    r = pyoracle.decode(g, llr[i].astype(np.float64), kind, kernel, i_max=imax, k_info=spec.k_info, n_p=4, log_cap=8000)
    ol = r["log_edge"]
    n = min(len(ol), 8000)
    gl = glog[i][:n]
    bad = np.flatnonzero(gl != ol[:n])
    lim = bad[0] if len(bad) else n
    vd = np.flatnonzero(gval[i][:lim] != r["log_c2v"][:lim])
    print(f"   committed values differ (before divergence) at steps {vd[:5].tolist()} of {lim}")
    if len(vd):
        k = vd[0]; print(f"   step {k}: oracle {r['log_c2v'][k]!r} gpu {gval[i][k]!r} edge {ol[k]}")
    print(f"frame {f}: oracle prop {r['prop']} gpu prop {int(out['prop'][i])}; first diff at step "
          f"{bad[0] if len(bad) else None}")
    if len(bad):
        k = bad[0]
        print("   oracle", ol[max(0,k-3):k+4].tolist(), "gap", r["log_gap"][k])
        print("   gpu   ", gl[max(0,k-3):k+4].tolist())
        print("   oracle gaps", r["log_gap"][max(0,k-3):k+4].tolist())
        print("   values oracle", r["log_c2v"][max(0,k-3):k+1].tolist(), "gpu", gval[i][max(0,k-3):k+1].tolist())
