"""Pick the tile width EB per (shape, order) from sweeps of every variant
library (tools/build_variants.sh).  Runs on the GPU box:

  python tools/tune_eb.py --variants 16,8,4,2,1 --ops helm > gpurun_out/tune.jsonl

Prints every measurement as a JSON line, then one line with the best EB per
(op, shape, order) and the kTunedEB table to paste into csrc/sk_tune.h.
"""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="op0_eb16,op0_eb8,op0_eb4,op0_eb2,op0_eb1")
    ap.add_argument("--ops", default="helm")
    ap.add_argument("--orders", default="1-10")
    ap.add_argument("--shapes", default="hex,prism,pyr,tet")
    ap.add_argument("--gbytes", default="1.0")
    ap.add_argument("--reps", default="8")
    ap.add_argument("--geo", default="deformed")
    a = ap.parse_args()
    best = {}
    for v in a.variants.split(","):
        lib = os.path.join(ROOT, "paper_2604_04644_b200", f"libsk200_{v}.so")
        kv = {t.rstrip("0123456789"): int(t[len(t.rstrip("0123456789")):]) for t in v.split("_")}
        nt_, mb_ = kv.get("nt", 0), kv.get("mb", -1)
        env = dict(os.environ, SK200_LIB=lib)
        cmd = [sys.executable, os.path.join(ROOT, "tools", "sweep.py"), "--ops", a.ops, "--orders", a.orders, "--shapes", a.shapes,
               "--gbytes", a.gbytes, "--reps", a.reps, "--geo", a.geo]
        out = subprocess.run(cmd, env=env, capture_output=True, text=True)
        if out.returncode:
            print(json.dumps({"variant": v, "error": out.stderr[-2000:]}), flush=True)
            continue
        for line in out.stdout.splitlines():
            rec = json.loads(line)
            rec["variant"] = v
            print(json.dumps(rec), flush=True)
            key = (rec["op"], rec["shape"], rec["P"])
            if key not in best or rec["gdof_s"] > best[key][1]:
                best[key] = ((rec["eb_nt_smem"][0], nt_, mb_), rec["gdof_s"], rec["roofline_frac"])
    shapes = ["hex", "prism", "pyr", "tet"]
    tables = {"kTunedEB": [[0] * 11 for _ in shapes], "kTunedNTDiv": [[1] * 11 for _ in shapes],
              "kTunedMinB": [[0] * 11 for _ in shapes]}
    for (op, s, P), ((eb, nt, mb), g, f) in sorted(best.items()):
        if op == "helm":
            tables["kTunedEB"][shapes.index(s)][P] = eb
            tables["kTunedNTDiv"][shapes.index(s)][P] = nt
            tables["kTunedMinB"][shapes.index(s)][P] = mb
    print(json.dumps({"best": {f"{k[0]}/{k[1]}/{k[2]}": v for k, v in sorted(best.items())}, **tables}))


if __name__ == "__main__":
    main()
