"""Trace one frame of a seeded batch (llr_batch) through GPU vs oracle logs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import pyoracle
from paper_2102_11089_b200.channel import llr_batch
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch_logged
from tests.util import load_code
key, kind, frame = sys.argv[1], sys.argv[2], int(sys.argv[3])
n_p = int(sys.argv[4]) if len(sys.argv) > 4 else 4
spec, g = load_code(key)
imax = {"C0": 5, "C1": 3, "C2": 3}[key]; eb = {"C0": 2.0, "C1": 2.0, "C2": 1.0}[key]
llr = llr_batch(spec, eb, 0, frame, 1)
cfg = ScheduleConfig(kind=kind, i_max=imax, n_p=n_p)
cap = imax * g.n_edges + n_p
out = decode_batch_logged(spec, torch.from_numpy(llr).cuda(), cfg, log_cap=cap)
gl = out["step_log"].cpu().numpy()[0]; gv = out["step_c2v"].cpu().numpy()[0]
r = pyoracle.decode(g, llr[0].astype(np.float64), kind, i_max=imax, k_info=spec.k_info, n_p=n_p, log_cap=cap)
ol, ov, og = r["log_edge"], r["log_c2v"], r["log_gap"]
n = min(len(ol), cap)
bad = np.flatnonzero(gl[:n] != ol[:n])
k = int(bad[0]) if len(bad) else None
print("first divergence", k, "of", n)
if k is not None:
    lo, hi = max(0, k - 6), k + 6
    print("oracle edges", ol[lo:hi].tolist()); print("  vns", g.edge_vn[ol[lo:hi]].tolist())
    print("gpu    edges", gl[lo:hi].tolist()); print("  vns", g.edge_vn[gl[lo:hi]].tolist())
    print("oracle gaps ", np.round(og[lo:hi], 6).tolist())
    vd = np.flatnonzero(gv[:k] != ov[:k])
    print("committed-value diffs before divergence:", len(vd), "max rel",
          float(np.max(np.abs(gv[vd] - ov[vd]) / np.abs(ov[vd]))) if len(vd) else 0)
