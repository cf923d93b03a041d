"""Compare roofline fractions of sweep JSONL files side by side:
  python tools/cmp_sweep.py old.jsonl new.jsonl [...]"""
import json
import sys

tabs = []
for f in sys.argv[1:]:
    d = {}
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        if "op" in r:
            d[(r["op"], r["shape"], r["P"])] = r
    tabs.append(d)
keys = sorted(set().union(*[t.keys() for t in tabs]), key=lambda k: (k[0], ["hex", "prism", "pyr", "tet"].index(k[1]), k[2]))
for k in keys:
    cells = []
    for t in tabs:
        r = t.get(k)
        cells.append(f"{r['roofline_frac']:.3f} ({r['gdof_s']:6.2f})" if r else " " * 15)
    print(f"{k[0]:6s} {k[1]:6s} P={k[2]:2d}  " + "   ".join(cells))
