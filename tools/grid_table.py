"""Print the tools/grid.py JSON lines as a table: python tools/grid_table.py profiles/r2/r2k_grid_*.jsonl"""
import json
import sys

for path in sys.argv[1:]:
    print("==", path)
    for l in open(path):
        r = json.loads(l)
        s = (f"{r['config']} {r['ebn0_db']:>4} dB B={r['batch']:<7} {r['schedule']:<14} {r['ms']:>10.1f} ms  "
             f"{r['frames_per_s']:>10.0f} fr/s {r['edge_updates_per_s']:.3e} upd/s {r['updates_per_frame']:>9.0f} upd/fr "
             f"FER {r['fer']:.4f} BER {r['ber_info']:.2e}")
        if "oracle_frames" in r:
            s += (f" | oracle n={r['oracle_frames']} FER {r['oracle_fer']:.4f} FER/BER in CI "
                  f"{int(r['fer_inside_ci95'])}/{int(r['ber_inside_ci95'])} identical "
                  f"{r['gpu_oracle_identical'][0]}/{r['gpu_oracle_identical'][1]} cpu {r['oracle_updates_per_s']:.2e} upd/s "
                  f"({r['oracle_cores']} cores)")
        print(s)
