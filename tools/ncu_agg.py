import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui=h.index('Metric Unit')
agg = collections.defaultdict(list)
for r in rows[hdr+1:]:
    if len(r) > vi:
        v = float(r[vi].replace(',','')); u = r[ui]
        v = v/1e3 if u in ('nsecond','ns') else (v*1e3 if u in ('msecond','ms') else v)
        agg[r[ki][:70]].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):9.1f} us {100*sum(v)/tot:5.1f}%  n={len(v):3d}  avg={sum(v)/len(v):8.2f}  {k}")
print("total us", tot)
