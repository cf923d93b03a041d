# C0 hex scatter over element-face patches (2) vs (x, z) tiles (1): assembly tests under 2, c0hex A/B, kernel time
SK_C0_SCATTER_TILED=2 timeout 900 python -m pytest tests -m gpu -q -k "c0 or C0 or assembl or multirank" 2>&1 | tail -1
for t in 1 2 1 2; do SK_C0_SCATTER_TILED=$t timeout 900 python bench.py --workload c0hex --sweep off > gpurun_out/r2run89_c0hex_$t.json 2>/dev/null; python3 -c "
import json; l=json.loads(open('gpurun_out/r2run89_c0hex_$t.json').read().strip().splitlines()[-1]); print('scatter=$t', round(l['value'],3), round(l['roofline']['frac'],3))"; done
mkdir -p gpurun_out/r2run89
SK_C0_SCATTER_TILED=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_c0" -c 2 --csv --log-file gpurun_out/r2run89/launches.csv python bench.py --workload c0hex --steps 2 --warmup 1 --sweep off > /dev/null 2>&1
grep -E "k_c0" gpurun_out/r2run89/launches.csv | awk -F'","' '{print $NF}' | head -2
