"""List the loops of a cuobjdump -sass function dump: backward branches, the
instruction count of each loop body and its opcode histogram."""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 50
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?)\s*;", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA (0x[0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            body = ins[addr[tgt]:i + 1]
            if len(body) < minlen:
                continue
            c = collections.Counter()
            for _, tt in body:
                op = re.sub(r"^@!?U?P\w+\s+", "", tt).split()[0].split(".")[0]
                c[op] += 1
            print(f"loop {hex(tgt)}..{hex(a)}: {len(body)} instr")
            print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common(24)))
