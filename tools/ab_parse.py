"""Summarise tools/ab_variants.sh output: best-of-reps microseconds per (case, kind, variant)."""
import collections
import json
import sys

d = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    tag, js = line.split(" ", 1)
    try:
        j = json.loads(js)
    except ValueError:
        continue
    v = tag[:-1]
    key = (j["case"], j["kind"].replace("prefix_prefill", "pp"))
    d[key][v] = min(d[key].get(v, 1e9), round(j["ms"] * 1000, 1))
vs = sorted({v for x in d.values() for v in x}, key=lambda v: (v != "a", v))
print("case | kind | " + " | ".join(vs))
for (c, k), x in d.items():
    print(f"{c} | {k} | " + " | ".join(str(x.get(v, "-")) for v in vs))
