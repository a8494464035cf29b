"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel (usage: ncu_launches.py CSV [top] [filter])."""
import csv,sys
from collections import defaultdict
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value'); iu=h.index('Metric Unit')
agg=defaultdict(lambda:[0,0.0]); seq=[]
for r in rows[1:]:
    try: v=float(r[iv].replace(',',''))
    except: continue
    if r[iu] in ('nsecond','ns'): v/=1e6
    elif r[iu] in ('usecond','us'): v/=1e3
    name=r[ik].split('(')[0].replace('void ','')[:70]
    agg[name][0]+=1; agg[name][1]+=v; seq.append((name,v))
print('total ms %.2f'%sum(v for _,v in seq))
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]:
    print('%-70s n=%4d  %.3f ms' % (k,n,t))
if len(sys.argv)>3:
    print([(n[:30], round(v,2)) for n,v in seq if sys.argv[3] in n])
