"""Per-source-line totals from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv, sys
rows, f, hdr = [], None, None
for r in csv.reader(open(sys.argv[1])):
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0] and r[0] != "Function Name":
        try: rows.append((f, int(r[0]), r[1][:90], int(r[4]), int(r[7])))
        except ValueError: pass
tot_s = sum(x[3] for x in rows); tot_i = sum(x[4] for x in rows)
key = 3 if len(sys.argv) < 3 else 4
print(f"total samples {tot_s} instr {tot_i}")
for x in sorted(rows, key=lambda x: -x[key])[:int(sys.argv[3]) if len(sys.argv) > 3 else 60]:
    print(f"{x[3]/tot_s*100:5.1f}% {x[4]/tot_i*100:5.1f}%i {x[0]}:{x[1]}  {x[2]}")
