"""Summarise an ncu launch list (CSV) and a full capture (.ncu-rep) into profiles/."""
import collections, csv, json, subprocess, sys
from pathlib import Path

def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    agg = collections.OrderedDict()
    scale = {"s": 1, "second": 1, "ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
        agg.setdefault(d["Kernel Name"], []).append(v)
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "seconds": sum(v), "share": sum(v) / tot} for k, v in agg.items()], tot

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__inst_executed.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio", "l1tex__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]

def capture_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for k, un, x in zip(h, u, v):
        if k in WANT or k == "Kernel Name":
            d[k] = (x, un)
    return d

if __name__ == "__main__":
    tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    shares, tot = launch_shares(launches)
    cap = capture_summary(rep)
    Path("profiles").mkdir(exist_ok=True)
    json.dump({"tag": tag, "launch_list": shares, "total_seconds": tot, "full_capture": cap},
              open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
    for s in shares:
        print(f"{s['launches']:3d} {s['seconds']:8.3f}s {100*s['share']:5.1f}%  {s['kernel'][:80]}")
    for k, (x, un) in cap.items():
        print(f"  {k} = {x} {un}")
