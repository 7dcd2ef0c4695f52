"""Median value per (bench args, library variant) from gpu_ab2.sh output."""
import json
import statistics
import sys
from collections import defaultdict

v = defaultdict(list)
order = []
for ln in open(sys.argv[1]):
    if not ln.startswith("{"):
        continue
    d = json.loads(ln)
    k = (d["args"], d["lib"])
    if k not in v:
        order.append(k)
    v[k].append(d["value"])
base = {}
for a, lib in order:
    m = statistics.median(v[(a, lib)])
    base.setdefault(a, m)
    print(f"{a[:44]:44s} {lib:10s} {m:.4e}  {m / base[a]:.4f}  (n={len(v[(a, lib)])}, "
          f"spread {(max(v[(a, lib)]) - min(v[(a, lib)])) / m * 100:.2f}%)")
