"""Attribute an ncu SASS-level capture to source lines (dev tool).

  ncu -i REP --page source --csv --print-source sass > sass.csv
  nvdisasm -gi KERNELS.cubin > dis.txt        (cubin: cuobjdump -xelf all libmlob.so)
  python tools/sass_lines.py sass.csv dis.txt KERNEL_SYMBOL [column] [top]

Joins the per-instruction metric column (default "Instructions Executed")
with nvdisasm's line table and prints the top source lines, both by the
innermost line and by the outermost call site in the kernel body."""
import collections
import csv
import re
import sys


def line_map(dis_path, sym):
    sec = f".text.{sym}:"
    out, cur, chain = {}, None, []
    on = False
    pat = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    ins = re.compile(r"^\s+/\*([0-9a-f]{4,6})\*/")
    with open(dis_path) as f:
        for ln in f:
            if ln.startswith(sec):
                on = True
                continue
            if on and ln.startswith("//----"):
                break
            if not on:
                continue
            m = pat.search(ln)
            if m:
                inner = (m.group(1).split("/")[-1], int(m.group(2)))
                if m.group(3):
                    chain.append(inner)
                    chain.append((m.group(3).split("/")[-1], int(m.group(4))))
                else:
                    if chain and chain[-1] == inner:
                        cur = (chain[0], inner)
                    else:
                        cur = (inner, inner)
                    chain = []
                continue
            m = ins.match(ln)
            if m and cur:
                out[int(m.group(1), 16)] = cur
    return out


def main():
    csv_path, dis_path, sym = sys.argv[1:4]
    col = sys.argv[4] if len(sys.argv) > 4 else "Instructions Executed"
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    lm = line_map(dis_path, sym)
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    ci = rows[hdr].index(col)
    base = None
    inner, outer = collections.Counter(), collections.Counter()
    total = 0.0
    for r in rows[hdr + 1:]:
        if not r or not r[0].startswith("0x"):
            continue
        a = int(r[0], 16)
        base = a if base is None else base
        v = float(r[ci] or 0)
        total += v
        loc = lm.get(a - base)
        if loc is None:
            continue
        inner[loc[0]] += v
        outer[loc[1]] += v
    print(f"{col}: total {total:.4g}")
    for name, c in (("innermost line", inner), ("kernel-body line", outer)):
        print(f"-- by {name}")
        for (fn, ln), v in c.most_common(top):
            print(f"{v / total * 100:6.2f}%  {fn}:{ln}")


if __name__ == "__main__":
    main()
