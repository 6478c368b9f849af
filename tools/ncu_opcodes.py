"""Warp-stall samples of an ncu report aggregated by SASS opcode and stall reason (ncu --page source, sass view).

    python tools/ncu_opcodes.py gpurun_out/prof.ncu-rep
"""
import csv, io, subprocess, sys, collections
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(out)))
hdr=rows[1]; data=rows[2:]
ix={h:i for i,h in enumerate(hdr)}
reasons=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
byop=collections.defaultdict(lambda: collections.Counter())
tot=collections.Counter()
execs=collections.Counter()
for r in data:
    if len(r)<len(hdr): continue
    op=r[ix['Source']].split()
    if not op: continue
    o=op[0]
    if o.startswith('@'): o=op[1]
    o=o.split('.')[0]
    for h in reasons:
        v=int(r[ix[h]] or 0); byop[o][h]+=v; tot[h]+=v
    execs[o]+=int(r[ix['Instructions Executed']] or 0)
T=sum(tot.values())
print('total samples',T)
for h,v in tot.most_common(): print(f'{h:22s} {100*v/T:5.1f}%')
print()
for o,c in sorted(byop.items(), key=lambda kv:-sum(kv[1].values()))[:18]:
    s=sum(c.values())
    print(f'{o:8s} {100*s/T:5.1f}%  exec {execs[o]/1e6:8.1f}M  ', ' '.join(f'{k[6:]}={100*v/T:.1f}' for k,v in c.most_common(4)))
