"""Instruction mix of the innermost backward-branch loops of a kernel's SASS
(development aid): python tools/sass_loop_mix.py OBJ MANGLED_NAME"""
import re
import subprocess
import sys
from collections import Counter

obj, fun = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, obj], capture_output=True, text=True).stdout
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)", txt)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr and i - addr[tgt] > 20:
            body = [t for _, t in ins[addr[tgt]:i + 1]]
            ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
            print(f"loop {hex(tgt)}..{hex(a)}: {len(body)} instrs")
            print("  ", ", ".join(f"{k} {v}" for k, v in ops.most_common(18)))
