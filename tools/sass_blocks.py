"""Basic blocks of a cuobjdump -sass listing, largest LOP3 blocks first, with
their opcode mix (diagnosis of the K2 step loop before spending GPU time).
usage: python tools/sass_blocks.py file.sass [n]"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for a, t in ins:
    for m in re.finditer(r"0x([0-9a-f]+)", t):
        if t.split()[0].lstrip("@!P0123456789T ").startswith(("BRA", "BSSY", "CALL", "JMP")) or " BRA " in t or t.startswith("BRA"):
            targets.add(int(m.group(1), 16))
blocks, cur = [], []
for a, t in ins:
    if a in targets and cur:
        blocks.append(cur); cur = []
    cur.append((a, t))
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    if op.startswith(("BRA", "EXIT", "RET", "BSYNC")):
        blocks.append(cur); cur = []
if cur:
    blocks.append(cur)
def opc(t):
    w = t.split()
    return w[1] if w[0].startswith("@") else w[0]
blocks.sort(key=lambda b: -sum(opc(t).startswith("LOP3") for _, t in b))
for b in blocks[:n]:
    c = Counter(opc(t) for _, t in b)
    alu = sum(v for k, v in c.items() if k.split(".")[0] in ("LOP3", "ISETP", "SEL", "IADD3", "LEA", "SHF", "PRMT", "PLOP3", "VIADD", "POPC", "FLO", "BREV", "VOTE", "MOV"))
    print(f"block @{b[0][0]:#x}: {len(b)} instrs, ALU-pipe-ish {alu}: " + ", ".join(f"{k} {v}" for k, v in c.most_common(14)))
