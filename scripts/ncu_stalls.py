"""Summarise an ncu --page source --print-source sass CSV: stall reasons overall
and per 100-instruction window (profiling helper, not product code)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ia = h.index('Instructions Executed')
isrc = h.index('Source')
sc = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
idx = {c: h.index(c) for c in sc}
tot = collections.Counter()
win = collections.defaultdict(collections.Counter)
W = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for j, r in enumerate(data):
    for c in sc:
        v = int(r[idx[c]] or 0)
        tot[c] += v
        win[j // W][c] += v
T = sum(tot.values())
print('total samples', T, 'instr', sum(int(r[ia] or 0) for r in data))
print(' '.join(f"{c[6:]}={v / T:.3f}" for c, v in tot.most_common(10)))
for w, cnt in sorted(win.items(), key=lambda x: -sum(x[1].values()))[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    s = sum(cnt.values())
    ops = collections.Counter()
    for k in range(w * W, min(w * W + W, len(data))):
        t = data[k][isrc].split()
        if t:
            ops[(t[1] if t[0].startswith('@') else t[0]).split('.')[0]] += 1
    print(f"{w * W:6d} {s / T:.3f} ", ' '.join(f"{c[6:]}={v / s:.2f}" for c, v in cnt.most_common(4)), '|',
          ' '.join(f"{o}:{n}" for o, n in ops.most_common(5)))
