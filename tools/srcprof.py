"""Aggregate ncu SASS-level stall samples per CUDA source line (via nvdisasm line info)."""
import csv, re, subprocess, sys, io
from collections import Counter, defaultdict
rep, cubin, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
isamp = h.index('Warp Stall Sampling (All Samples)')
iexe = h.index('Instructions Executed')
stalls = [i for i, k in enumerate(h) if k.startswith('stall_') and 'Not Issued' not in k]
sass = rows[2:]
dis = subprocess.run(['nvdisasm', '--print-line-info', cubin], capture_output=True, text=True).stdout
parts = re.split(r'\n\s*\.text\.(\S+):', dis)
body = None
for i in range(1, len(parts), 2):
    if fn in parts[i]:
        body = parts[i + 1]
        break
lines = []
cur = None
for x in body.split('\n'):
    m = re.search(r'//## File "([^"]+)", line (\d+)', x)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    if re.search(r'/\*[0-9a-f]{4,}\*/', x):
        lines.append(cur)
print('sass rows', len(sass), 'disasm instrs', len(lines), file=sys.stderr)
agg = Counter(); st = defaultdict(Counter); ex = Counter()
tot = 0
for i, r in enumerate(sass):
    if i >= len(lines):
        break
    s = int(r[isamp] or 0)
    tot += s
    agg[lines[i]] += s
    ex[lines[i]] += int(r[iexe] or 0)
    for j in stalls:
        v = int(r[j] or 0)
        if v:
            st[lines[i]][h[j][6:]] += v
src = {}
for (f, ln), s in agg.most_common(top):
    top3 = ', '.join(f'{k}:{100*v/s:.0f}%' for k, v in st[(f, ln)].most_common(3)) if s else ''
    print(f'{100*s/tot:5.1f}%  {f}:{ln}  inst={ex[(f,ln)]:>11}  {top3}')
