import collections,sys
d=collections.defaultdict(list)
for l in open(sys.argv[1]):
    if l.startswith("KLOG"):
        _,k,c,f,fr,us=l.split(); d[(int(k),int(c),int(f))].append(float(us))
names=["K1","K2P","K2C","K3P","K3C","plan"]
rows=sorted(d.items(), key=lambda x:(x[0][0],x[0][1]))
tot=sum(sum(v) for v in d.values())
for (k,c,f),v in rows:
    print(f"{names[k]:4s} cells={c:8d} faces={f:8d} n={len(v):3d} avg_us={sum(v)/len(v):8.2f} ns/cell={sum(v)/len(v)*1e3/max(c,1):6.3f} share={sum(v)/tot:.3f}")
