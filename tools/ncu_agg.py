import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
h=rows[0]; rows=rows[1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    t=float(r[vi].replace(',',''))/1e6
    name=r[ki].split('(')[0]
    agg[name][0]+=1; agg[name][1]+=t
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{v[1]:8.3f} ms {v[0]:5d}  {k[:90]}")
print("total", tot, len(rows))
