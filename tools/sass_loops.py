"""List the loops of a SASS dump (backward branches) with their instruction mix.
    cuobjdump -sass -fun <mangled> obj.o > k.sass; python tools/sass_loops.py k.sass"""
import re
import sys
from collections import Counter

ins = []
for line in open(sys.argv[1]):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
for i, (addr, txt) in enumerate(ins):
    m = re.search(r"\bBRA(?:\.\S+)?\s+(?:\S+,\s*)?0x([0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= addr:
        continue
    body = [t for a, t in ins if tgt <= a <= addr]
    c = Counter()
    for t in body:
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        c[op.split(".")[0]] += 1
    if c["LDS"] == 0 and c["LDG"] == 0:
        continue
    print(f"loop 0x{tgt:x}-0x{addr:x}: {len(body)} instr, LDS {c['LDS']}, LDG {c['LDG']}, SHFL {c['SHFL']}, "
          f"per-LDS {len(body) / max(c['LDS'], 1):.2f}")
    print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common(18)))
