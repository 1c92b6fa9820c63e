"""Benchmark: decoded frames/s and C2V edge updates/s per schedule (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C0|C1|C2|C3|C4|C3F]

Workload (default): BASELINE.json configs[1] -- the WiFi-shaped n=648 QC code
(Z=27), BPSK-AWGN at Eb/N0 = 2.0 dB (mid-sweep), i_max = 3, batch 100,000
frames, float64 (the reference's arithmetic), and every schedule the config
names (flooding, layered, RBP, CIRBP, LMDRBP, sLMDRBP, LMD-CIRBP, ME-CIRBP
M=4, ME-RBP M=4).  One step = the batch decoded once by every schedule.
value = total C2V edge updates / time over the K timed steps (whole job, all
ranks).  The batch's LLRs (259 MB) exceed the 126 MB L2, so every step
streams its inputs from HBM.

The same run also measures BASELINE configs[3] -- the largest single-GPU
config, the BG1-shaped n=26112 code (Z=384, 2Z punctured) at 1.0 dB, i_max 10,
10,000 frames, flooding / layered / RBP / CIRBP / ME-CIRBP M=64 -- as the
`secondary.C3` block with its own roofline, CPU legs and GPU==oracle identity
(1 warm-up + 1 timed step: one C3 step is minutes of GPU time, so the driver's
20 + 5 steps of it would not fit its time limit; `--workload C3` runs it as
the main line).

--impl reference: the reference's OWN decoder (ldpc_ids.schedules.decode,
numba, installed unmodified in baseline/_ref) on all host cores through the
reference harness's process-pool pattern (sim.py:233-259), same config and
metric, each step a bounded seeded sample of the batch (one frame per core);
layered (absent from the reference) runs on the C port (oracle/ldpc_oracle.c).
Without baseline/_ref the C port runs every schedule.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (config key, ebn0, i_max, batch, [(kind, n_p)])
    "C1": ("C1", 2.0, 3, 100_000,
           [("flooding", 1), ("layered", 1), ("rbp", 1), ("cirbp", 1), ("lmdrbp", 1), ("slmdrbp", 1),
            ("lmd_cirbp", 1), ("me_cirbp", 4), ("me_rbp", 4)]),
    "C0": ("C0", 2.0, 5, 10_000, [("flooding", 1), ("layered", 1), ("rbp", 1), ("cirbp", 1)]),
    "C2": ("C2", 1.0, 3, 100_000, [("layered", 1), ("rbp", 1), ("cirbp", 1), ("me_cirbp", 1),
                                   ("me_cirbp", 4), ("me_cirbp", 16)]),
    "C3": ("C3", 1.0, 10, 10_000, [("flooding", 1), ("layered", 1), ("rbp", 1), ("cirbp", 1),
                                   ("me_cirbp", 64)]),
    "C3b": ("C3", 0.5, 10, 10_000, [("flooding", 1), ("layered", 1), ("rbp", 1), ("cirbp", 1),
                                    ("me_cirbp", 64)]),
    # C4 = the C2 code at 0 dB, budget 20 E (batch/occupancy sweep: --batch)
    "C4": ("C2", 0.0, 20, 16_384, [("me_cirbp", 1), ("me_cirbp", 4), ("me_cirbp", 16), ("me_cirbp", 64),
                                   ("rbp", 1)]),
    # BG1 fixed schedules only (the roofline case: HBM-bound frame-interleaved kernels)
    "C3F": ("C3", 1.0, 10, 10_000, [("flooding", 1), ("layered", 1)]),
}

CI_KINDS = {"cirbp", "lmd_cirbp", "me_cirbp", "me_lmd_cirbp"}
# random 32-byte-sector read bandwidth of HBM at a >= 4 GB footprint, measured on the pool's
# B200s with tools/micro/randbw (profiles/r2/r2m_random_sector_bandwidth.json)
RANDOM_SECTOR_GBPS = 1170.0


def bytes_per_update(kind, counters, E, N, elem):
    """Algorithmic message-state bytes per C2V update,
    in units of the state element size `elem` (4 = fp32 figures, 8 = fp64)."""
    s = elem / 4.0
    P = max(1, int(counters[:, 0].sum()))
    if kind == "flooding":
        return s * (16 + 8 * N / E)
    if kind == "layered":
        return s * 16
    V, R, I = (int(counters[:, k].sum()) for k in (1, 2, 3))
    base = 20 + (8 if kind in CI_KINDS else 0)
    return s * (base + (12 * V + 28 * R + 8 * I) / P)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup(args):
    import torch
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() and args.impl == "ours" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available() and args.impl == "ours":
        torch.cuda.set_device(local)
    return rank, world, local


def make_inputs(spec, ebn0, start, count):
    from paper_2102_11089_b200.channel import llr_batch
    return llr_batch(spec, ebn0, seed=0, start=start, count=count, dtype=np.float32)


def _sname(kind, n_p):
    return kind + (f"/M{n_p}" if kind.startswith("me_") else "")


def run_reference(args, wl):
    """The reference's own decoder on all host cores; rank 0 only (the other
    ranks exit without work)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    from oracle import pyoracle, refpool
    from paper_2102_11089_b200 import configs
    from paper_2102_11089_b200.codes import build_tanner
    key, ebn0, i_max, batch, scheds = wl
    spec = getattr(configs, f"make_{key.lower()}_code")()
    g = build_tanner(spec.h)
    cores = os.cpu_count() or 1
    # one frame per core per step for the BG1-shaped code (seconds of CPU per
    # frame), 2048 frames otherwise (the same order of CPU time per step)
    sample = args.ref_sample or (cores if key == "C3" else min(batch, 2048))
    llr = make_inputs(spec, ebn0, 0, sample).astype(np.float64)
    use_ref = refpool.available() and not args.ref_port
    pool = refpool.RefPool(spec, scheds, i_max, workers=cores) if use_ref else None
    ref_kinds = set(pool.scheds) if pool else set()
    port = [(k, n) for k, n in scheds if (k, n) not in ref_kinds]

    def step():
        t0 = time.perf_counter()
        upd = 0
        if pool:
            r, _ = pool.run(llr)
            upd += sum(v[0] for v in r.values())
        for kind, n_p in port:
            r = pyoracle.decode_batch(g, llr, kind, i_max=i_max, k_info=spec.k_info, n_p=n_p, threads=cores)
            upd += int(r["prop"].sum())
        return upd, time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    tot_u = tot_t = 0
    for _ in range(args.steps):
        u, t = step()
        tot_u += u
        tot_t += t
    if pool:
        pool.close()
    val = tot_u / tot_t
    what = ("ldpc_ids.schedules.decode (numba, baseline/_ref) over a %d-process pool (sim.py:233-259)"
            % cores if pool else "C port oracle/ldpc_oracle.c, %d threads" % cores)
    if pool and port:
        what += "; " + ", ".join(_sname(k, n) for k, n in port) + " (not in the reference) on the C port"
    line = {
        "impl": "reference", "metric": f"C2V edge updates/s (all {args.workload} schedules); decoded frames/s",
        "value": val, "unit": "C2V edge updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "frames_per_s": sample * len(scheds) * args.steps / tot_t,
        "config": {"workload": f"{args.workload} ({spec.label}): " + ", ".join(_sname(k, n) for k, n in scheds),
                   "code": spec.label, "ebn0_db": ebn0, "i_max": i_max, "batch": sample},
        "cpu_baseline": {"value": val, "unit": "C2V edge updates/s", "cores": cores,
                         "kind": "reference" if pool else "port",
                         "sample": f"first {sample} frames of the seeded batch per step, every schedule: {what}"},
        "e2e": {"value": val, "unit": "C2V edge updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(wl, spec, g, llr_host, gpu_outs, budget_s=20.0):
    """C port (oracle/ldpc_oracle.c) on a bounded sample of the same batch, all
    host cores (rank 0, N=1 only): first one frame per core through every
    schedule, then, if that took less than the budget, a larger sample scaled
    to ~budget_s.  Also reports, per schedule, the fraction of sample frames on
    which the GPU's decode of the same frames (gpu_outs) is identical to the
    oracle's (hard decisions and update count)."""
    from oracle import pyoracle
    key, ebn0, i_max, batch, scheds = wl
    cores = os.cpu_count() or 1

    def run(sample):
        per, tot_u = {}, 0
        t0 = time.perf_counter()
        for si, (kind, n_p) in enumerate(scheds):
            t1 = time.perf_counter()
            r = pyoracle.decode_batch(g, sample, kind, i_max=i_max, k_info=spec.k_info, n_p=n_p,
                                      threads=cores)
            u = int(r["prop"].sum())
            n = len(sample)
            gu = gpu_outs[si]["u_hat"][:n].cpu().numpy()
            gp = gpu_outs[si]["prop"][:n].cpu().numpy()
            same = (gu == r["u_hat"]).all(1) & (gp == r["prop"])
            per[_sname(kind, n_p)] = {"updates_per_s": u / (time.perf_counter() - t1),
                                      "frame_errors": int((r["bit_errors_at"][:, -1] > 0).sum()),
                                      "bit_errors": int(r["info_bit_errors_at"][:, -1].sum()),
                                      "bits": r["info_bit_errors_at"][:, -1].copy(),
                                      "frames": n, "identical": int(same.sum())}
            tot_u += u
        return tot_u, time.perf_counter() - t0, per

    n = min(len(llr_host), cores)
    u, t, per = run(llr_host[:n].astype(np.float64))
    if t < budget_s / 2 and n < len(llr_host):
        n = int(min(len(llr_host), max(n, n * budget_s / max(t, 1e-3)) // cores * cores))
        u, t, per = run(llr_host[:n].astype(np.float64))
    return {"value": u / t, "unit": "C2V edge updates/s", "cores": cores, "kind": "port",
            "sample": f"first {n} frames of the batch through every schedule ({t:.1f} s)",
            "frames_per_s": n * len(scheds) / t,
            "per_schedule_updates_per_s": {k: v["updates_per_s"] for k, v in per.items()},
            "per_schedule_fer": {k: (v["frame_errors"], v["frames"]) for k, v in per.items()},
            "per_schedule_info_bits": {k: v["bits"] for k, v in per.items()},
            "gpu_oracle_identical": {k: [v["identical"], v["frames"]] for k, v in per.items()}}


def cpu_reference(wl, spec, llr_host, budget_s=30.0):
    """The reference's own numba decoder (baseline/_ref) over the harness's
    process pool on the first frames of the batch: the `--impl reference` leg,
    reported beside the C port (rank 0, N=1 only)."""
    from oracle import refpool
    if not refpool.available():
        return None
    key, ebn0, i_max, batch, scheds = wl
    cores = os.cpu_count() or 1
    pool = refpool.RefPool(spec, scheds, i_max, workers=cores)
    try:
        n = cores
        r, t = pool.run(llr_host[:n])
        if t < budget_s / 2:
            n = int(min(len(llr_host), max(n, n * budget_s / max(t, 1e-3)) // cores * cores))
            r, t = pool.run(llr_host[:n])
    finally:
        pool.close()
    u = sum(v[0] for v in r.values())
    return {"value": u / t, "unit": "C2V edge updates/s", "cores": cores, "kind": "reference",
            "sample": f"first {n} frames, schedules {', '.join(_sname(k, m) for k, m in r)} through "
                      f"ldpc_ids.schedules.decode (numba) on a {cores}-process pool ({t:.1f} s)",
            "per_schedule_updates_per_s": {_sname(k, m): v[0] / t * len(r) for (k, m), v in r.items()},
            "per_schedule_fer": {_sname(k, m): (v[1], n) for (k, m), v in r.items()}}


def ber_ci(bits_per_frame, k_info, alpha=0.05, reps=2000, seed=0):
    """95 % interval of the info-bit error rate from per-frame bit-error counts:
    percentile bootstrap over frames (bit errors cluster in erroneous frames,
    so a binomial over bits would be far too narrow)."""
    b = np.asarray(bits_per_frame, np.float64)
    n = len(b)
    if n == 0:
        return 0.0, 1.0
    rng = np.random.default_rng(seed)
    means = b[rng.integers(0, n, size=(reps, n))].mean(1)
    lo, hi = np.quantile(means, [alpha / 2, 1 - alpha / 2])
    if b.sum() == 0:  # no error in the sample: BER <= FER <= 3/n (rule of three)
        return 0.0, 3.0 / n
    return float(lo) / k_info, float(hi) / k_info


def _json_default(o):
    """numpy scalars / arrays that reach the JSON line as plain Python values."""
    if isinstance(o, np.ndarray):
        return o.tolist()
    if isinstance(o, np.generic):
        return o.item()
    raise TypeError(f"Object of type {o.__class__.__name__} is not JSON serializable")


def clopper_pearson(k, n, alpha=0.05):
    """Exact two-sided binomial confidence interval (FER CI, north star)."""
    from scipy.stats import beta
    lo = 0.0 if k == 0 else float(beta.ppf(alpha / 2, k, n - k + 1))
    hi = 1.0 if k == n else float(beta.ppf(1 - alpha / 2, k + 1, n - k))
    return lo, hi


def run_ours(args, wl):
    rank, world, local = dist_setup(args)
    cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
    line = measure(args, wl, args.workload, args.steps, args.warmup, rank, world, local,
                   batch=args.batch, cpu=cpu)
    if args.workload == "C1" and not args.no_secondary and not args.only:
        # BASELINE configs[3] (C3, the BG1-shaped code at 10k frames) on the same
        # clock: one step is minutes of GPU time, so 1 warm-up + 1 timed step
        sec = measure(args, WORKLOADS["C3"], "C3", 1, 1, rank, world, local, batch=0, cpu=cpu, e2e=False)
        line["secondary"] = {"C3": {k: sec[k] for k in sec if k not in ("e2e",)}}
        if args.secondary_f32:
            # the same C3 block with float32 state (the north star's GPU arithmetic: half the
            # sectors per update; parity there is 1e-4 on message values, not bit identity)
            import copy
            a32 = copy.copy(args)
            a32.precision = "f32"
            s32 = measure(a32, WORKLOADS["C3"], "C3", 1, 1, rank, world, local, batch=0, cpu=False, e2e=False)
            line["secondary"]["C3_f32"] = {k: s32[k] for k in s32 if k not in ("e2e",)}
    if rank == 0:
        print(json.dumps(line, default=_json_default), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def measure(args, wl, wname, steps, warmup, rank, world, local, batch=0, cpu=False, e2e=True):
    import torch
    from paper_2102_11089_b200 import configs
    from paper_2102_11089_b200 import dist as D
    from paper_2102_11089_b200.codes import build_tanner
    from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch, device_graph

    key, ebn0, i_max, wl_batch, scheds = wl
    batch = batch or wl_batch
    if args.only:
        scheds = [s for s in scheds if s[0] + (f"/M{s[1]}" if s[0].startswith("me_") else "") == args.only]
        if not scheds:
            raise SystemExit(f"--only {args.only}: not a schedule of {key}")
    spec = getattr(configs, f"make_{key.lower()}_code")()
    g = build_tanner(spec.h)
    dg = device_graph(g)
    E, N = g.n_edges, g.n_vars
    elem = 8 if args.precision == "f64" else 4
    dev = torch.device("cuda", torch.cuda.current_device())
    start, _ = D.shard(batch, rank)  # weak scaling: disjoint frame-index ranges per rank
    llr_host = make_inputs(spec, ebn0, start, batch)
    llr_pinned = torch.from_numpy(llr_host).pin_memory()
    llr_dev = llr_pinned.to(dev)
    cfgs = [ScheduleConfig(kind=k, i_max=i_max, n_p=n_p, precision=args.precision) for k, n_p in scheds]
    stream = torch.cuda.current_stream(dev)
    outs = {}

    def one(cfg, idx, src):
        outs[idx] = decode_batch(g, src, cfg, k_info=spec.k_info, out=outs.get(idx))
        return outs[idx]["_launches"]

    # warm-up (also yields the per-schedule work, identical every step)
    for _ in range(max(1, warmup)):
        for i, c in enumerate(cfgs):
            one(c, i, llr_dev)
    torch.cuda.synchronize()
    work = []
    for i, c in enumerate(cfgs):
        cnt = outs[i]["counters"].cpu().numpy()
        fer = float((outs[i]["bit_errors_at"][:, -1] > 0).float().mean().item())
        ber = float(outs[i]["info_bit_errors_at"][:, -1].double().sum().item()) / (batch * max(1, spec.k_info))
        work.append({"updates": int(cnt[:, 0].sum()), "bpu": bytes_per_update(c.kind, cnt, E, N, elem),
                     "fer": fer, "ber": ber, "counters": cnt.sum(0)})

    # timed region: device-resident inputs
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in cfgs] for _ in range(steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches = 0
    t_start.record(stream)
    for s in range(steps):
        for i, c in enumerate(cfgs):
            ev[s][i][0].record(stream)
            launches += one(c, i, llr_dev)
            ev[s][i][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    sched_ms = [sum(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(steps)) / steps
                for i in range(len(cfgs))]

    # e2e: pinned host LLRs in, host results out, through the public API
    res_host = {i: {k: torch.empty_like(outs[i][k], device="cpu").pin_memory()
                    for k in ("u_hat", "prop", "converged")} for i in range(len(cfgs))}
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e_start.record(stream)
    h2d = d2h = 0
    for s in range(steps if e2e else 0):
        src = llr_pinned.to(dev, non_blocking=True)
        h2d += llr_pinned.numel() * llr_pinned.element_size()
        for i, c in enumerate(cfgs):
            one(c, i, src)
            for k in ("u_hat", "prop", "converged"):
                res_host[i][k].copy_(outs[i][k], non_blocking=True)
                d2h += outs[i][k].numel() * outs[i][k].element_size()
    e_end.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e_start.elapsed_time(e_end)

    step_updates = int(D.all_sum([sum(w["updates"] for w in work)])[0])  # all ranks
    t_max, e_max = (float(x) for x in D.all_max([total_ms, e2e_ms]))
    job_updates = step_updates * steps
    value = job_updates / (t_max / 1e3)
    e2e_value = job_updates / (e_max / 1e3) if e2e else None

    # dominant kernel roofline (algorithmic state bytes / kernel time)
    dom = int(np.argmax(sched_ms))
    w = work[dom]
    achieved = w["updates"] * w["bpu"] / (sched_ms[dom] / 1e3) / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # DRAM traffic of this kernel from a committed ncu --set full capture of
    # `bench.py --only <kernel>` (profiles/traffic.json), per launch
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    dom_name = cfgs[dom].kind + (f"/M{cfgs[dom].n_p}" if cfgs[dom].kind.startswith("me_") else "")
    if tf.exists():
        tj = json.loads(tf.read_text())
        t = tj.get(f"{key}:{dom_name}:{args.precision}:{batch}")
        traffic = t.get("dram_bytes_per_launch") if t else None
        if traffic is None:
            # no capture of this exact launch: a per-update figure measured on the same code,
            # schedule and placement at full occupancy (ncu dram bytes / updates) x this launch's updates
            t = tj.get(f"{key}:{dom_name}:{args.precision}:per_update")
            traffic = t["dram_bytes_per_update"] * work[dom]["updates"] if t else None
    per = {}
    for i, (c, wk) in enumerate(zip(cfgs, work)):
        nm = c.kind + (f"/M{c.n_p}" if c.kind.startswith("me_") else "")
        per[nm] = {"ms": round(sched_ms[i], 3), "edge_updates_per_s": wk["updates"] / (sched_ms[i] / 1e3),
                   "frames_per_s": batch / (sched_ms[i] / 1e3), "fer": wk["fer"], "ber_info": wk["ber"],
                   "updates_per_frame": wk["updates"] / batch, "state_bytes_per_update": round(wk["bpu"], 1),
                   "state_GBps": wk["updates"] * wk["bpu"] / (sched_ms[i] / 1e3) / 1e9}
    line = {
        "metric": f"C2V edge updates/s (all {wname} schedules); decoded frames/s",
        "value": value, "unit": "C2V edge updates/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": t_max / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "frames_per_s": batch * len(cfgs) * steps * world / (t_max / 1e3),
        "config": {"workload": f"{wname} ({spec.label}): " + ", ".join(f"{k}(n_p={n})" for k, n in scheds),
                   "code": spec.label, "N": N, "E": E, "ebn0_db": ebn0, "i_max": i_max,
                   "batch_per_gpu": batch, "l2": "inputs > L2 (batch LLRs %.0f MB)" % (llr_pinned.numel() * 4 / 1e6),
                   "parallelism": f"frames sharded over {world} GPU(s)"},
        "per_schedule": per,
        "roofline": {"bound": "hbm", "kernel": list(per)[dom], "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src,
                     # the dynamic schedules touch scattered 32-byte sectors of a multi-GB state:
                     # the HBM figure that bounds them is the random-sector rate measured by
                     # tools/micro/randbw (profiles/r2/r2m_random_sector_bandwidth.json), not the copy rate
                     "random_sector_peak": RANDOM_SECTOR_GBPS,
                     "dram_rate": (traffic / (sched_ms[dom] / 1e3) / 1e9) if traffic else None,
                     "dram_rate_vs_random_sector_peak":
                         (traffic / (sched_ms[dom] / 1e3) / 1e9 / RANDOM_SECTOR_GBPS) if traffic else None,
                     "note": "achieved = algorithmic message-state bytes per launch (SURVEY 8(d) "
                             "formula in %s units x the launch's C2V updates) / the launch's CUDA-event "
                             "time; peak = HBM copy bandwidth.  The dynamic schedules read and write "
                             "scattered sectors (8 useful bytes per 32-byte sector for the per-VN words), "
                             "so their DRAM traffic (`traffic`, ncu) is 3-5x the algorithmic bytes and the "
                             "bound that applies is the random-sector rate (`random_sector_peak`, GB/s "
                             "of 32-byte sectors at >= 4 GB footprint)" % args.precision},
        "e2e": {"value": e2e_value, "unit": "C2V edge updates/s", "h2d_bytes_per_step": h2d // steps,
                "d2h_bytes_per_step": d2h // steps} if e2e else None,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if cpu:
        cb = cpu_baseline(wl, spec, g, llr_host, [outs[i] for i in range(len(cfgs))], budget_s=args.cpu_budget)
        line["cpu_baseline"] = cb
        for nm, (same, n) in cb["gpu_oracle_identical"].items():
            if nm in per:
                per[nm]["gpu_oracle_identical"] = [same, n]
        cr = cpu_reference(wl, spec, llr_host, budget_s=args.cpu_budget)
        if cr:
            line["cpu_reference"] = cr
        # FER vs oracle: the GPU's FER over the whole batch must lie inside the
        # oracle sample's 95 % Clopper-Pearson interval (north star)
        for nm, (k, n) in cb["per_schedule_fer"].items():
            if nm in per:
                lo, hi = clopper_pearson(k, n)
                per[nm]["oracle_fer_sample"] = k / n
                per[nm]["oracle_fer_ci95"] = [lo, hi]
                per[nm]["fer_inside_oracle_ci95"] = bool(lo <= per[nm]["fer"] <= hi)
        # BER (info bits): frame-level bootstrap interval of the sample's rate
        for nm, bits in cb.pop("per_schedule_info_bits").items():
            if nm in per:
                k = max(1, spec.k_info)
                lo, hi = ber_ci(bits, k)
                per[nm]["oracle_ber_sample"] = float(np.mean(bits)) / k
                per[nm]["oracle_ber_ci95"] = [lo, hi]
                per[nm]["ber_inside_oracle_ci95"] = bool(lo <= per[nm]["ber_info"] <= hi)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C1", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--ref-port", action="store_true", help="reference arm on the C port even if baseline/_ref exists")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C3 block of the default C1 run")
    ap.add_argument("--secondary-f32", action="store_true", help="also run the C3 block with float32 state")
    ap.add_argument("--only", default="", help="run one schedule of the workload (e.g. cirbp, me_rbp/M4)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours" and not os.environ.get("BENCH_ALLOW_SHORT"):
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
