"""BASELINE.json config grid on the GPU, with the CPU oracle beside it.

    python tools/grid.py PART [--out FILE]

PART selects a slice of the grid (so each gpurun call stays bounded):
  c0      configs[0]: C0 at 2.0 dB, 10k frames, flooding/layered/RBP/CIRBP, i_max 5
  c1      configs[1]: C1 at 1.0..3.0 dB, 100k frames, all single-edge + ME-CIRBP/ME-RBP M=4
  c2      configs[2]: C2 at 0.5..2.0 dB, 100k frames, layered/RBP/CIRBP/ME-CIRBP M=1,4,16
  c3      configs[3]: C3 at 0.5 and 1.0 dB, 10k frames, flooding/layered/RBP/CIRBP/ME-CIRBP M=64
  c4      configs[4]: C2 code at 0 dB, i_max 20, batches 1..16k (all five schedules), 256k (two)
  c4m     configs[4]: the 1M-frame batch, ME-CIRBP(64)

One JSON line per (config, SNR, schedule, batch): GPU time (CUDA events, one
untimed warm-up decode of up to 8192 frames first), frames/s, C2V updates/s, FER and info-BER over
the whole batch; the oracle (oracle/ldpc_oracle.c, all host cores) on the
first S frames of the same batch: its FER / BER with 95 % intervals
(Clopper-Pearson for FER; a frame-level bootstrap for BER, bit errors cluster),
whether the GPU's values fall inside them, and the fraction of those S frames
the GPU decoded identically (hard decisions and update count).
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import pyoracle  # noqa: E402
from paper_2102_11089_b200 import configs  # noqa: E402
from paper_2102_11089_b200.channel import llr_batch  # noqa: E402
from paper_2102_11089_b200.codes import build_tanner  # noqa: E402
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch  # noqa: E402

C1S = [("flooding", 1), ("layered", 1), ("rbp", 1), ("cirbp", 1), ("lmdrbp", 1), ("slmdrbp", 1),
       ("lmd_cirbp", 1), ("me_cirbp", 4), ("me_rbp", 4)]
C2S = [("layered", 1), ("rbp", 1), ("cirbp", 1), ("me_cirbp", 1), ("me_cirbp", 4), ("me_cirbp", 16)]
C3S = [("flooding", 1), ("layered", 1), ("rbp", 1), ("cirbp", 1), ("me_cirbp", 64)]
C4S = [("me_cirbp", 1), ("me_cirbp", 4), ("me_cirbp", 16), ("me_cirbp", 64), ("rbp", 1)]
PARTS = {
    "c0": [("C0", eb, 5, 10_000, [("flooding", 1), ("layered", 1), ("rbp", 1), ("cirbp", 1)], 2000) for eb in (2.0,)],
    "c1": [("C1", eb, 3, 100_000, C1S, 1000 if eb < 2.5 else 4000) for eb in (1.0, 1.5, 2.0, 2.5, 3.0)],
    "c2": [("C2", eb, 3, 100_000, C2S, 256) for eb in (0.5, 1.0, 1.5, 2.0)],
    "c3": [("C3", eb, 10, 10_000, C3S, 32) for eb in (0.5, 1.0)],
    "c4": [("C4", 0.0, 20, b, C4S, 0) for b in (1, 64, 1024, 16384)] +
          [("C4", 0.0, 20, 262_144, [("me_cirbp", 64), ("rbp", 1)], 0)],
    "c4m": [("C4", 0.0, 20, 1_048_576, [("me_cirbp", 64)], 0)],  # the 1M-frame point (about 15 GPU-minutes)
    "c4r": [("C4", 0.0, 20, 1_048_576, [("rbp", 1)], 0)],
}


def code_of(key):
    return configs.make_c2_code() if key == "C4" else getattr(configs, f"make_{key.lower()}_code")()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("part", choices=sorted(PARTS))
    ap.add_argument("--out", default="")
    ap.add_argument("--precision", default="f64")
    args = ap.parse_args()
    out = open(args.out, "a") if args.out else sys.stdout
    cores = os.cpu_count() or 1
    for key, eb, i_max, B, scheds, S in PARTS[args.part]:
        spec = code_of(key)
        g = build_tanner(spec.h)
        llr_h = llr_batch(spec, eb, seed=0, start=0, count=B)
        llr = torch.from_numpy(llr_h).cuda()
        for kind, n_p in scheds:
            cfg = ScheduleConfig(kind=kind, i_max=i_max, n_p=n_p, precision=args.precision)
            # warm-up on a bounded slice (kernel load, device graph, workspace);
            # the timed decode's outputs are allocated first, outside the events
            o = decode_batch(spec, llr[:min(B, 8192)], cfg)
            o = {k: torch.zeros((B,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device) for k, v in o.items() if torch.is_tensor(v)}
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            o = decode_batch(spec, llr, cfg, out=o)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            upd = int(o["prop"].sum().item())
            fe = int((o["bit_errors_at"][:, -1] > 0).sum().item())
            be = float(o["info_bit_errors_at"][:, -1].double().sum().item())
            k = max(1, spec.k_info)
            row = {"config": key, "code": spec.label, "ebn0_db": eb, "i_max": i_max, "batch": B,
                   "schedule": bench._sname(kind, n_p), "precision": args.precision, "ms": round(ms, 3),
                   "frames_per_s": B / (ms / 1e3), "edge_updates_per_s": upd / (ms / 1e3),
                   "updates_per_frame": upd / B, "fer": fe / B, "ber_info": be / (B * k)}
            if S:
                n = min(S, B)
                t0 = time.perf_counter()
                r = pyoracle.decode_batch(g, llr_h[:n].astype(np.float64), kind, i_max=i_max, k_info=spec.k_info,
                                          n_p=n_p, threads=cores)
                dt = time.perf_counter() - t0
                ofe = int((r["bit_errors_at"][:, -1] > 0).sum())
                lo, hi = bench.clopper_pearson(ofe, n)
                bits = r["info_bit_errors_at"][:, -1].astype(np.float64)
                blo, bhi = bench.ber_ci(bits, k)
                gu = o["u_hat"][:n].cpu().numpy()
                gp = o["prop"][:n].cpu().numpy()
                same = (gu == r["u_hat"]).all(1) & (gp == r["prop"])
                row.update({"oracle_frames": n, "oracle_fer": ofe / n, "oracle_fer_ci95": [lo, hi],
                            "fer_inside_ci95": bool(lo <= row["fer"] <= hi),
                            "oracle_ber_info": bits.mean() / k, "oracle_ber_ci95": [blo, bhi],
                            "ber_inside_ci95": bool(blo <= row["ber_info"] <= bhi),
                            "gpu_oracle_identical": [int(same.sum()), n],
                            "oracle_updates_per_s": int(r["prop"].sum()) / dt, "oracle_cores": cores})
            out.write(json.dumps(row) + "\n")
            out.flush()
        del llr


if __name__ == "__main__":
    main()
