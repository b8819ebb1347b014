"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per
CUDA source line (profiling helper, not product code).
usage: ncu_lines.py export.csv [file-substring] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else "nsw_step_kernel"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur = None
hdr = None
per = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] and cur and want in cur:
        d = dict(zip(hdr, r))
        try:
            per.append((int(d["Warp Stall Sampling (All Samples)"] or 0), int(d["Instructions Executed"] or 0),
                        int(r[0]), r[1].strip()[:90]))
        except (ValueError, KeyError):
            pass
tot = sum(p[0] for p in per) or 1
toti = sum(p[1] for p in per) or 1
print(f"file~{want}: samples {tot} instr {toti}")
for s, i, ln, src in sorted(per, reverse=True)[:top]:
    print(f"{ln:5d} {s / tot:6.3f} {i / toti:6.3f}  {src}")
