"""Instruction / stall share per enclosing device function (ncu source CSV with
--print-source cuda,sass).  usage: funcshare.py CSV"""
import csv, re, sys, collections
srcs = {}
def fn_map(path):
    if path in srcs: return srcs[path]
    m = {}; cur = '?'
    try:
        for i, l in enumerate(open(path), 1):
            g = re.search(r'(?:__device__|__global__)[^(]*?\b(\w+)\s*\(', l)
            if g and not l.strip().startswith('//'): cur = g.group(1)
            m[i] = cur
    except OSError: pass
    srcs[path] = m; return m
agg = collections.Counter(); st = collections.Counter(); f = None; ii = ws = None
for r in csv.reader(open(sys.argv[1])):
    if not r: continue
    if r[0] in ("File Path", "File Name"): f = r[1]; continue
    if r[0] == "Line No": ii = r.index("Instructions Executed"); ws = r.index("Warp Stall Sampling (All Samples)"); continue
    if ii is None or not r[0].isdigit(): continue  # source rows only (SASS rows have no line)
    try: n = float(r[ii] or 0); s = float(r[ws] or 0)
    except ValueError: continue
    key = f.split('/')[-1] + ':' + fn_map(f).get(int(r[0]), '?')
    agg[key] += n; st[key] += s
tn = sum(agg.values()); ts = sum(st.values())
for k, v in agg.most_common(40): print(f"{v/tn*100:5.1f}%i {st[k]/ts*100:5.1f}%s  {k}")
