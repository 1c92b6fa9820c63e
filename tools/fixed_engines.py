"""Time flooding / layered under each fixed engine (ldpc_sched_t.variant = phase |
tile | pipe) on the bench codes, to set the engine-choice heuristic.

    python tools/fixed_engines.py [C0,C1,C2,C3] [f64,f32] [phase,tile,pipe] [tag]
Prints one JSON line per (code, precision, kind, engine).
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

CASES = {"C0": (2.0, 5, 10_000), "C1": (2.0, 3, 100_000), "C2": (1.0, 3, 100_000), "C3": (1.0, 10, 10_000)}
codes = sys.argv[1].split(",") if len(sys.argv) > 1 else list(CASES)
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["f64", "f32"]
engines = sys.argv[3].split(",") if len(sys.argv) > 3 else ["phase", "tile", "pipe"]
tag = sys.argv[4] if len(sys.argv) > 4 else ""
for key in codes:
    eb, imax, B = CASES[key]
    spec = getattr(configs, f"make_{key.lower()}_code")()
    g = build_tanner(spec.h)
    llr = torch.from_numpy(llr_batch(spec, eb, 0, 0, B)).cuda()
    for prec in precs:
        for kind in ("flooding", "layered"):
            cfg = ScheduleConfig(kind=kind, i_max=imax, precision=prec)
            for eng in engines:
                var = {"phase": "fixed_phase", "tile": "fixed_tile", "pipe": "fixed_pipe"}[eng]
                out = None
                for _ in range(2):
                    out = decode_batch(g, llr, cfg, k_info=spec.k_info, out=out, variant=var)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(3):
                    out = decode_batch(g, llr, cfg, k_info=spec.k_info, out=out, variant=var)
                b.record()
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / 3
                upd = int(out["prop"].sum())
                print(json.dumps({"tag": tag, "code": key, "prec": prec, "kind": kind, "engine": eng, "ms": round(ms, 3),
                                  "upd_per_s": upd / ms * 1e3}), flush=True)
