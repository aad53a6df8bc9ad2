"""Summarise an ncu source page (sass, csv): stall reasons by instruction class
and the top stalled instructions.  usage: ncu_stalls.py page.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[idx['Source']].strip()
    op = src.split()[0] if src else ''
    if op.startswith('@'):
        op = src.split()[1]
    op = op.split('.')[0]
    s = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    lines.append((s, r[idx['Address']], src[:70], {h: int(r[idx[h]] or 0) for h in stalls}))
    for h in stalls:
        v = int(r[idx[h]] or 0)
        tot[h] += v
        byop[op][h] += v
T = sum(tot.values())
print("total samples", T)
for h, v in tot.most_common(10):
    print(f"  {h:28s} {100 * v / T:5.1f}%")
print("by opcode:")
for op, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    s = sum(c.values())
    print(f"  {op:10s} {100 * s / T:5.1f}%  " + ", ".join(f"{k[6:]}={100 * v / T:.1f}" for k, v in c.most_common(3)))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("top instructions:")
for s, a, src, d in sorted(lines, key=lambda x: -x[0])[:top]:
    best = sorted(d.items(), key=lambda kv: -kv[1])[:2]
    print(f"  {a} {100 * s / T:5.1f}% {src:70s} " + ", ".join(f"{k[6:]}={v}" for k, v in best))
