import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
tot=collections.defaultdict(float); cnt=collections.Counter()
for r in rows[1:]:
    try: v=float(r[vi].replace(',',''))
    except: continue
    name=r[ki][:70]; tot[name]+=v; cnt[name]+=1
T=sum(tot.values())
for n,v in sorted(tot.items(), key=lambda x:-x[1])[:int(sys.argv[2]) if len(sys.argv)>2 else 22]: print(f"{v/T*100:6.2f}% {v/cnt[n]/1e3:9.1f} us x{cnt[n]:4d} {n}")
print(T/1e6, 'ms total')
