"""Per-instruction stall samples of one SASS loop from an ncu source-page CSV
(--page source --csv --print-source sass): prints the loop in windows with
samples and dominant stall reasons (profiling helper, not product code).
usage: python scripts/ncu_loop_profile.py CSV MIN_FFMA [window]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
isrc, iadr = h.index('Source'), h.index('Address')
ismp = h.index('Warp Stall Sampling (All Samples)')
iex = h.index('Instructions Executed')
sc = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
ix = {c: h.index(c) for c in sc}
ins = [(int(r[iadr], 16), r[isrc].strip(), r) for r in data]
addr = {a: i for i, (a, _, _) in enumerate(ins)}
minf = int(sys.argv[2])
W = int(sys.argv[3]) if len(sys.argv) > 3 else 40
loops = []
for i, (a, s, _) in enumerate(ins):
    m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)", s)
    if m:
        t = int(m.group(1), 16)
        if t <= a and t in addr:
            body = ins[addr[t]:i + 1]
            nf = sum(1 for _, x, _ in body if 'FFMA' in x)
            if nf >= minf:
                loops.append((addr[t], i))
allT = sum(int(r[ismp] or 0) for _, _, r in ins)
for lo, hi in loops:
    body = ins[lo:hi + 1]
    T = sum(int(r[ismp] or 0) for _, _, r in body)
    print(f"== loop {ins[lo][0]:#x}-{ins[hi][0]:#x}: {hi - lo + 1} instr, {T} samples ({T / allT:.1%} of kernel)")
    for w0 in range(0, len(body), W):
        seg = body[w0:w0 + W]
        st = collections.Counter()
        for _, _, r in seg:
            for c in sc:
                st[c[6:]] += int(r[ix[c]] or 0)
        n = sum(st.values())
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for _, x, _ in seg if x)
        print(f" [{w0:4d}] {n:6d} ({n / max(T, 1):5.1%}) " + " ".join(f"{k}={v}" for k, v in st.most_common(4)) +
              " | " + " ".join(f"{k}{v}" for k, v in ops.most_common(5)))
