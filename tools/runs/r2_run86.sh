# mapped C0 scatter / gather without 64-bit divisions (W == 1): assembly tests + bench
timeout 900 python -m pytest tests -m gpu -q -k "c0 or C0 or assembl or multirank" 2>&1 | tail -1
for w in c0prism c0tet c0pyr c0hex; do timeout 900 python bench.py --workload $w --sweep off > gpurun_out/r2run86_$w.json 2>/dev/null; python3 -c "
import json; l=json.loads(open('gpurun_out/r2run86_$w.json').read().strip().splitlines()[-1]); print('$w', round(l['value'],3), round(l['roofline']['frac'],3), round(l['e2e']['value'],3))"; done
