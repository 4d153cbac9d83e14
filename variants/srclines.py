"""Per-source-line totals from `ncu -i X --page source --csv --print-source cuda,sass`.
usage: srclines.py CSV [column-name] [top-n]"""
import csv, sys
col = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows, f, idx, ii = [], None, None, None
for r in csv.reader(open(sys.argv[1])):
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": idx = r.index(col); ii = r.index("Instructions Executed"); continue
    if idx and r[0] and r[0] not in ("Function Name", "Kernel Name"):
        try: rows.append((f, int(r[0]), r[1][:90], float(r[idx] or 0), float(r[ii] or 0)))
        except ValueError: pass
tot = sum(x[3] for x in rows) or 1; toti = sum(x[4] for x in rows) or 1
print(f"column {col}: total {tot:.0f}; instructions {toti:.3e}")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[3]/tot*100:5.1f}% {x[4]/toti*100:5.1f}%i {x[0]}:{x[1]}  {x[2]}")
