"""Stall reasons per code region (groups of SASS instructions with equal execution counts) from an
`ncu --page source --csv` export: which role of a warp-specialised kernel waits on what."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
grp = collections.defaultdict(lambda: [0, 0.0, collections.Counter(), collections.Counter()])
for r in rows[2:]:
    try:
        e = float(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    if e < float(sys.argv[2] if len(sys.argv) > 2 else 1e5):
        continue
    key = round(e / 1e4)
    g = grp[key]
    g[0] += 1
    g[1] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for s in stalls:
        g[2][s[6:]] += float(r[ix[s]] or 0)
    src = r[ix["Source"]]
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
    g[3][op] += 1
tot = sum(g[1] for g in grp.values())
for k in sorted(grp, key=lambda k: -grp[k][1])[:8]:
    g = grp[k]
    top = ", ".join(f"{s} {v / max(g[1], 1):.0%}" for s, v in g[2].most_common(6) if v > 0)
    print(f"exec {k / 100:6.2f}M x {g[0]:4d} instr  samples {g[1] / tot:5.1%}  [{top}]  ops {dict(g[3].most_common(8))}")
