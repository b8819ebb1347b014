"""List the loops of one kernel's SASS (backward branches) with their
instruction mix -- a build-time check of the hot loops (not product code).
usage: python scripts/sass_loops.py <cubin> <mangled-name-substring> [min_len]"""
import collections
import re
import subprocess
import sys

cubin, pat = sys.argv[1], sys.argv[2]
minlen = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0]
    if pat not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print("==", name[:110], len(ins), "instructions")
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)", t)
        if m and "BRA" in t:
            tgt = int(m.group(1), 16)
            if tgt <= a and tgt in addr and i - addr[tgt] >= minlen:
                body = [x for _, x in ins[addr[tgt]:i + 1]]
                ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for x in body)
                print(f"  loop 0x{tgt:x}-0x{a:x}: {len(body)} instr  " +
                      " ".join(f"{k}={v}" for k, v in ops.most_common(14)))
