"""Tabulate GDOF/s per (op, shape, P) across the variants of a tune_eb.py log:
  python tools/cmp_variants.py log.jsonl"""
import json
import sys

d, vs = {}, []
for line in open(sys.argv[1]):
    if not line.startswith('{"op"'):
        continue
    r = json.loads(line)
    v = r["variant"]
    if v not in vs:
        vs.append(v)
    d.setdefault((r["op"], r["shape"], r["P"]), {})[v] = r["gdof_s"]
print("op shape P " + " ".join(f"{v:>14s}" for v in vs))
for k, row in sorted(d.items()):
    base = row.get(vs[0])
    cells = []
    for v in vs:
        g = row.get(v)
        cells.append(f"{g:7.2f}({g / base:4.2f})" if g and base else f"{'-':>14s}")
    print(f"{k[0]} {k[1]:5s} {k[2]:2d} " + " ".join(cells))
