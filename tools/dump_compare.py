"""Compare GPU vs oracle ci / pre_total right before update `step` of one frame."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes as C
import numpy as np, torch
from oracle import pyoracle
from paper_2102_11089_b200 import _native
from paper_2102_11089_b200.channel import llr_batch
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch
from tests.util import load_code
key, kind, frame, steps = sys.argv[1], sys.argv[2], int(sys.argv[3]), [int(x) for x in sys.argv[4].split(",")]
spec, g = load_code(key)
imax = {"C0": 5, "C1": 3, "C2": 3}[key]; eb = {"C0": 2.0, "C1": 2.0, "C2": 1.0}[key]
llr = llr_batch(spec, eb, 0, frame, 1)
cfg = ScheduleConfig(kind=kind, i_max=imax, n_p=4)
L = _native.lib()
for st in steps:
    buf = torch.zeros(2 * g.n_vars + 8192 + 2 * g.n_edges, dtype=torch.float64, device="cuda")
    L.ldpc_set_state_dump(st, C.c_void_p(buf.data_ptr()))
    decode_batch(spec, torch.from_numpy(llr).cuda(), cfg); torch.cuda.synchronize()
    L.ldpc_set_state_dump(-1, None)
    gb = buf.cpu().numpy()
    r = pyoracle.decode_dump(g, llr[0].astype(np.float64), st, kind=kind, i_max=imax, k_info=spec.k_info, n_p=4)
    dci = np.flatnonzero(gb[:g.n_vars] != r["dump_ci"]); dpt = np.flatnonzero(gb[g.n_vars:2 * g.n_vars] != r["dump_pretot"])
    rel = np.max(np.abs(gb[:g.n_vars] - r["dump_ci"]) / np.maximum(np.abs(r["dump_ci"]), 1e-300)) if len(dci) else 0
    print(f"step {st}: ci differs at {len(dci)} VNs (max rel {rel:.3g}), pre_total at {len(dpt)} VNs;",
          "first", dci[:5].tolist(), [ (r['dump_ci'][n], gb[n]) for n in dci[:3]])
    ng = 16
    go = np.minimum((r["dump_ci"] * ng).astype(np.int64), ng - 1)
    gg = np.minimum((gb[:g.n_vars] * ng).astype(np.int64), ng - 1)
    d = np.flatnonzero(go != gg)
    print("   group differences:", d.tolist(), [(r["dump_ci"][n] * ng, gb[n] * ng) for n in d[:4]])
    x = r["dump_ci"] * ng
    rr = np.floor(x + 0.5)
    m = (rr >= 1) & (rr <= ng - 1)
    print("   min rel boundary distance (oracle ci):", float(np.min(np.abs(x[m] - rr[m]) / rr[m])) if m.any() else None)
    grng = gb[2 * g.n_vars:2 * g.n_vars + 8192].view(np.int64)[:len(r["rng_log"])]
    dr = np.flatnonzero(grng != r["rng_log"])
    print("   rng states:", len(r["rng_log"]), "first differing selection:", dr[:3].tolist(),
          (r["rng_log"][dr[0]], grng[dr[0]]) if len(dr) else "")
    o = 2 * g.n_vars + 8192
    gpre, gc2v = gb[o:o + g.n_edges], gb[o + g.n_edges:o + 2 * g.n_edges]
    for name, a, b in (("pre", r["dump_pre"], gpre), ("c2v", r["dump_c2v"], gc2v)):
        rel = np.abs(a - b) / np.maximum(np.abs(a), 1e-30)
        big = np.flatnonzero(rel > 1e-9)
        print(f"   {name}: {int((a != b).sum())} differ, {len(big)} by >1e-9 rel; worst", big[:6].tolist(),
              [(a[e], b[e]) for e in big[:3]])
    if len(sys.argv) > 5:
        n = int(sys.argv[5])
        es = g.vn_edges[g.vn_ptr[n]:g.vn_ptr[n + 1]]
        print("   VN", n, "edges", es.tolist(), "res oracle", np.abs(r["dump_pre"][es] - r["dump_c2v"][es]).tolist(),
              "gpu", np.abs(gpre[es] - gc2v[es]).tolist())
