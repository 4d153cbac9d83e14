"""Diagnostic: attribute ncu source-page samples / executed instructions of
step_kernel<4> to source lines (needs nvdisasm -g of the same binary)."""
import re, collections, csv, sys
dis, src = sys.argv[1], sys.argv[2]
cur = None; fn = None; off2line = {}
for l in open(dis):
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m: fn = m.group(1); continue
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m2 = re.search(r'/\*([0-9a-f]{4,6})\*/', l)
    if fn and 'step_kernelILi4' in fn and m2: off2line[int(m2.group(1), 16)] = cur
rows = list(csv.reader(open(src))); hdr = rows[1]; data = rows[2:]
ia = hdr.index('Address'); iss = hdr.index('Warp Stall Sampling (All Samples)'); iex = hdr.index('Instructions Executed')
base = int(data[0][ia], 16)
S = collections.Counter(); X = collections.Counter()
for r in data:
    k = off2line.get(int(r[ia], 16) - base)
    S[k] += float(r[iss] or 0); X[k] += float(r[iex] or 0)
ts, tx = sum(S.values()), sum(X.values())
files = {f: open(f'/root/repo/paper_2511_02136_b200/csrc/{f}').read().split('\n') for f in ('mlob_step.cuh', 'mlob_kernels.cu')}
key = sys.argv[3] if len(sys.argv) > 3 else 'exec'
top = (X if key == 'exec' else S).most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 50)
print(f"total exec {tx:.3e}  samples {ts:.0f}")
for k, v in top:
    txt = files[k[0]][k[1] - 1].strip()[:64] if k and k[0] in files else ''
    print(f"x{X[k]/tx*100:5.2f}% s{S[k]/ts*100:5.2f}% {k[0][:12] if k else None}:{k[1] if k else ''} {txt}")
