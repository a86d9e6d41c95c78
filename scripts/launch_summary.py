"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: launch_summary.py LIST.csv [TOP] [--ours]   (--ours: only this library's kernels, i.e. the
oid / k1tc / k1p / k1f / a9q / bgtc namespaces; block generation and torch glue outside the timed region dropped)"""
import csv, collections, sys
args = [a for a in sys.argv[1:] if not a.startswith("--")]
ours = "--ours" in sys.argv
rows = [r for r in csv.reader(open(args[0])) if len(r) > 5]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    try: v = float(r[vi].replace(',', ''))
    except ValueError: continue
    name = r[ki]
    if ours and not any(t in name for t in ("oid::", "k1tc::", "k1p::", "k1f::", "a9q::", "bgtc::")): continue
    name = name[:70]; tot[name] += v; cnt[name] += 1
T = sum(tot.values())
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:int(args[1]) if len(args) > 1 else 22]:
    print(f"{v/T*100:6.2f}% {v/cnt[n]/1e3:9.1f} us x{cnt[n]:4d} {n}")
print(T/1e6, 'ms total', '(this library only)' if ours else '')
