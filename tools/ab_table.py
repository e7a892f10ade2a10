"""Best-of-reps table of an abn.sh / ab.sh log: python tools/ab_table.py <log> [variants...]"""
import collections
import re
import sys

res = collections.defaultdict(dict)
order = []
for line in open(sys.argv[1]):
    m = re.match(r'(\w+?)(\d) \{"kind": "(prefix_prefill\w*)", "case": "([^"]+)", "ms": ([0-9.]+)', line)
    if not m:
        continue
    v, _, kind, case, ms = m.groups()
    if kind == "prefix_prefill_rope_contig_q":
        continue
    if v not in order:
        order.append(v)
    k = (case, kind)
    res[k][v] = min(res[k].get(v, 1e9), float(ms) * 1000)
vs = sys.argv[2:] or order
print(f"{'case':32s} {'kind':5s} " + " ".join(f"{v:>8s}" for v in vs) + "   (us, best of reps)")
for (case, kind), d in res.items():
    base = d.get(vs[0])
    cells = []
    for v in vs:
        x = d.get(v)
        cells.append(f"{x:8.1f}" if x else "       -")
    print(f"{case[:32]:32s} {kind[15:] or 'plain':5s} " + " ".join(cells))
