"""Resident-frame / placement sweep for the dynamic engine (sets the dyn_plan policy).

    python tools/dyn_sweep.py CODE KINDS [B] [f64|f32] [placements] [fractions]
KINDS: comma list, ME kinds as me_cirbp/4.  For each kind, placement in
auto/split/trees/hbm and max_resident in {auto, 1/4, 1/2, 3/4 of auto}:
one JSON line with ms and updates/s.
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2102_11089_b200 import configs  # noqa: E402
from paper_2102_11089_b200.channel import llr_batch  # noqa: E402
from paper_2102_11089_b200.codes import build_tanner  # noqa: E402
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch  # noqa: E402

EB = {"C0": (2.0, 5), "C1": (2.0, 3), "C2": (1.0, 3), "C3": (1.0, 10), "C4": (0.0, 20)}
key = sys.argv[1]
kinds = sys.argv[2].split(",")
B = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000
prec = sys.argv[4] if len(sys.argv) > 4 else "f64"
PLACES = sys.argv[5].split(",") if len(sys.argv) > 5 else ["auto", "split", "trees", "hbm"]
FRACS = [float(x) for x in sys.argv[6].split(",")] if len(sys.argv) > 6 else [0, 0.25, 0.5, 0.75]
VARIANTS = sys.argv[7].split(",") if len(sys.argv) > 7 else [""]
eb, imax = EB[key]
spec = getattr(configs, f"make_{'c2' if key == 'C4' else key.lower()}_code")()
g = build_tanner(spec.h)
llr = torch.from_numpy(llr_batch(spec, eb, 0, 0, B)).cuda()


def timed(cfg, **kw):
    out = decode_batch(g, llr, cfg, k_info=spec.k_info, **kw)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = decode_batch(g, llr, cfg, k_info=spec.k_info, out=out, **kw)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return ms, int(out["prop"].sum())


for ks in kinds:
    kind, _, m = ks.partition("/")
    cfg = ScheduleConfig(kind=kind, i_max=imax, n_p=int(m or 1), precision=prec)
    for pl, var in [(a, b) for a in PLACES for b in VARIANTS]:
        for frac in FRACS:
            res = 0
            if frac:
                res = max(32, int(frac * min(B, 148 * 64)))
            try:
                ms, upd = timed(cfg, placement=pl, max_resident=res, variant=var)
            except Exception as e:  # unsupported placement for this kind/code
                print(json.dumps({"kind": ks, "placement": pl, "res": res, "error": str(e)[:80]}), flush=True)
                break
            print(json.dumps({"lib": os.environ.get("LDPC_B200_LIB", "default")[-12:], "code": key, "kind": ks, "placement": pl, "variant": var, "res": res, "ms": round(ms, 2),
                              "upd_per_s": upd / ms * 1e3}), flush=True)
