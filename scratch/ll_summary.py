import csv,collections,sys
rows=[r for r in csv.reader(open(sys.argv[1] if len(sys.argv)>1 else '/root/repo/gpurun_out/launches_ll.csv')) if len(r)>10]
h=rows[0]
ki=h.index('Kernel Name'); ni=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
by=collections.defaultdict(dict)
for r in rows[1:]:
    by[(r[ii],r[ki][:60])][r[ni]]=float(r[vi].replace(',',''))
agg=collections.defaultdict(lambda: collections.defaultdict(float)); cnt=collections.Counter()
for (i,k),m in by.items():
    cnt[k]+=1
    for a,b in m.items(): agg[k][a]+=b
tot=sum(agg[k]['gpu__time_duration.sum'] for k in agg)
for k in sorted(agg,key=lambda k:-agg[k]['gpu__time_duration.sum'])[:int(sys.argv[2]) if len(sys.argv)>2 else 14]:
    m=agg[k]; c=cnt[k]
    print(f"{m['gpu__time_duration.sum']/tot*100:5.1f}% {m['gpu__time_duration.sum']/c/1e3:8.1f}us x{c:3d} inst {m.get('smsp__inst_executed.sum',0)/c/1e6:8.1f}M occ {m.get('sm__warps_active.avg.pct_of_peak_sustained_active',0)/c:5.1f}% thr/inst {m.get('smsp__thread_inst_executed_per_inst_executed.ratio',0)/c:5.1f} {k}")
