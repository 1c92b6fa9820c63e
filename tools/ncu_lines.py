"""Aggregate an ncu source page (--print-source cuda,sass CSV) per CUDA line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; data = []; hdr = None
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try: s = int(r[4]); ie = int(r[7])
        except Exception: continue
        data.append((s, ie, fname, r[0], r[1][:100]))
tot = sum(x[0] for x in data) or 1; tie = sum(x[1] for x in data) or 1
print("samples", tot, "instructions", tie)
for x in sorted(data, reverse=True)[:top]:
    print(f"{100*x[0]/tot:5.1f}%s {100*x[1]/tie:5.1f}%i {x[2]}:{x[3]} {x[4]}")
