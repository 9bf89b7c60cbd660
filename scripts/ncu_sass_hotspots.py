"""Per-SASS-opcode instruction counts (per point) and the top stalled SASS instructions of one
kernel in an ncu report.   python scripts/ncu_sass_hotspots.py <report> <kernel-regex> [n_points]
"""
import csv, sys, collections, subprocess
rep = sys.argv[1]; kern = sys.argv[2] if len(sys.argv)>2 else None
args=['ncu','-i',rep,'--page','source','--csv','--print-source','sass']
if kern: args+=['--kernel-name','regex:'+kern]
raw = subprocess.run(args,capture_output=True,text=True).stdout
r=list(csv.reader(raw.splitlines()))
h=r[1]; rows=[]
for x in r[2:]:
    if x and x[0]=='Kernel Name': break
    if len(x)==len(h): rows.append(x)
iS=h.index('Source'); iE=h.index('Instructions Executed'); iW=h.index('Warp Stall Sampling (All Samples)'); iA=h.index('Address')
f=lambda v: int(v.replace(',','') or 0)
tot=sum(f(x[iE]) for x in rows); totw=sum(f(x[iW]) for x in rows)
print('instr', tot, 'samples', totw)
c=collections.Counter(); s=collections.Counter()
for x in rows:
    t=x[iS].split()
    if not t: continue
    op=t[1] if t[0].startswith('@') else t[0]
    op=op.split('.')[0]
    c[op]+=f(x[iE]); s[op]+=f(x[iW])
npts=float(sys.argv[3]) if len(sys.argv)>3 else 7e6
for op,v in c.most_common(30): print('%-10s %8.1f/pt  stall %5.1f%%'%(op,v/npts,100*s[op]/totw))
print('--- top stall instructions')
for x in sorted(rows,key=lambda x:-f(x[iW]))[:25]:
    print('%5.1f%% %s %s  exec=%d'%(100*f(x[iW])/totw, x[iA], x[iS][:70], f(x[iE])))
