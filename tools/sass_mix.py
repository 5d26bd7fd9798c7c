"""Instruction mix of one kernel's hottest loop in a cuobjdump -sass listing.

Usage: python tools/sass_mix.py <lib.so|cubin> <kernel-name-substring>
Finds the function, then the innermost backward branch with the largest body
(the mainloop) and prints the opcode histogram of that body.
"""
import re
import subprocess
import sys
from collections import Counter

lib, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", txt)
body = None
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat in name:
        body = f
        print("function:", name)
        break
if body is None:
    sys.exit("not found")
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# backward branches
best = None
for addr, txt_ in ins:
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt_)
    tgt = None
    mm = re.search(r"0x([0-9a-f]+)", txt_)
    if "BRA" in txt_ and mm:
        tgt = int(mm.group(1), 16)
    if tgt is not None and tgt < addr:
        n = sum(1 for a, _ in ins if tgt <= a <= addr)
        if best is None or n > best[2]:
            best = (tgt, addr, n)
if best is None:
    sys.exit("no loop")
tgt, end, n = best
ops = Counter()
for a, t in ins:
    if tgt <= a <= end:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        ops[op.split(".")[0]] += 1
print(f"loop {tgt:#x}-{end:#x}: {n} instructions")
for op, c in ops.most_common():
    print(f"{c:6d} {op}")
