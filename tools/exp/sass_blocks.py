"""Basic blocks of one kernel's SASS (cuobjdump -sass) with instruction-class counts.
usage: python tools/exp/sass_blocks.py LIB.so KERNEL_SUBSTRING [min_block_len]"""
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
minlen = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
f = [x for x in funcs if pat in x.split("\n", 1)[0]]
if not f:
    sys.exit("kernel not found")
ins = []
for line in f[0].splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
targets = {int(m.group(1), 16) for _, t in ins for m in [re.search(r"BRA.*?0x([0-9a-f]+)", t)] if m}
blocks, cur = [], []
for a, t in ins:
    if a in targets and cur:
        blocks.append(cur)
        cur = []
    cur.append((a, t))
    if "BRA" in t or "EXIT" in t:
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
print(f"{len(ins)} instructions, {len(blocks)} blocks")
cls = {"dadd": "DADD", "dmul": "DMUL", "shfl": "SHFL", "ldg": "LDG", "stg": "STG", "ldl": "LDL", "stl": "STL",
       "lds": "LDS", "bar": "BAR"}
for b in blocks:
    n = len(b)
    c = {k: sum(v in t for _, t in b) for k, v in cls.items()}
    mov = sum(re.match(r"(@\S+ )?(MOV|IMAD.MOV)", t) is not None for _, t in b)
    if n >= minlen or c["ldl"] or c["stl"]:
        print(hex(b[0][0]), n, " ".join(f"{k}={v}" for k, v in c.items() if v), f"mov={mov}", "|", b[-1][1][:50])
