"""Pick the best variant per (op, shape, P) from tune JSONL files and print
the winners with their margin over a reference sweep.

  python tools/pick_tune.py --ref sweep.jsonl tune_a.jsonl tune_b.jsonl [--op helm]
"""
import argparse
import collections
import json

ap = argparse.ArgumentParser()
ap.add_argument("files", nargs="+")
ap.add_argument("--ref", default=None)
ap.add_argument("--op", default=None)
a = ap.parse_args()
res = collections.defaultdict(dict)
for f in a.files:
    for line in open(f):
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        if "op" not in r or "variant" not in r:
            continue
        if a.op and r["op"] != a.op:
            continue
        res[(r["op"], r["shape"], r["P"])][r["variant"]] = r["roofline_frac"]
ref = {}
if a.ref:
    for line in open(a.ref):
        if line.startswith("{"):
            r = json.loads(line)
            if "op" in r:
                ref[(r["op"], r["shape"], r["P"])] = r["roofline_frac"]
for k in sorted(res, key=lambda k: (k[0], ["hex", "prism", "pyr", "tet"].index(k[1]), k[2])):
    vs = res[k]
    ranked = sorted(vs.items(), key=lambda kv: -kv[1])
    rf = ref.get(k)
    print(f"{k[0]:5s} {k[1]:5s} P={k[2]:2d}  ref {rf if rf is None else round(rf, 3)}  "
          + "  ".join(f"{v}:{x:.3f}" for v, x in ranked[:4]))
