"""Summarise an `ncu --page source --csv --print-source sass` dump: top stall lines."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
to_i = lambda x: int(x) if x.strip().isdigit() else 0
tot = sum(to_i(r[i_s]) for r in data)
print("total samples", tot, "warp-instrs", sum(to_i(r[i_ex]) for r in data))
ops = {}
for r in data:
    op = r[i_src].split()[0] if r[i_src].split() else "?"
    if op.startswith("@"):
        op = r[i_src].split()[1]
    op = op.split(".")[0]
    ops[op] = ops.get(op, 0) + to_i(r[i_ex])
print("instr mix:", sorted(ops.items(), key=lambda kv: -kv[1])[:16])
for r in sorted(data, key=lambda r: -to_i(r[i_s]))[:n]:
    print(f"{to_i(r[i_s]):6d} {r[0][-5:]} {r[i_src][:100]}")
