"""Summarise an `ncu --page source --csv --print-source sass` export: stall samples by reason and by opcode.
usage: python tools/ncu_source_stalls.py SRC.csv"""
import csv,sys,collections,re
rows=list(csv.reader(open(sys.argv[1])))
name=rows[0][1]; hdr=rows[1]; data=rows[2:]
print(name[:90])
ix={h:i for i,h in enumerate(hdr)}
stalls=[h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot=collections.Counter(); byop=collections.defaultdict(collections.Counter); samples=0
for r in data:
    if len(r)<len(hdr): continue
    src=r[ix["Source"]].strip()
    op=re.sub(r"^@!?U?P\w+\s+","",src).split(" ")[0].split(".")[0]
    for s in stalls:
        v=int(r[ix[s]] or 0); tot[s]+=v; byop[op][s]+=v
T=sum(tot.values())
print("total samples",T)
for s,v in tot.most_common(12): print(f"  {s:28s} {v/T*100:5.1f}%")
print("by opcode (share of all samples; top stalls):")
ops=sorted(byop,key=lambda o:-sum(byop[o].values()))
for o in ops[:14]:
    t=sum(byop[o].values())
    print(f"  {o:10s} {t/T*100:5.1f}%  "+", ".join(f"{k[6:]} {v/T*100:.1f}" for k,v in byop[o].most_common(4)))
