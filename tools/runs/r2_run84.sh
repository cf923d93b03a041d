# C0 hex scatter over element-column tiles A/B (1: (x,z) tiles, 2: element-column tiles); assembly tests under both
for t in 2 1; do SK_C0_SCATTER_TILED=$t timeout 900 python -m pytest tests -m gpu -q -k "c0 or C0 or assembl or multirank" 2>&1 | tail -1; done
for t in 1 2 1 2; do SK_C0_SCATTER_TILED=$t timeout 900 python bench.py --workload c0hex --sweep off > gpurun_out/r2run84_c0hex_$t.json 2>/dev/null; python3 -c "
import json; l=json.loads(open('gpurun_out/r2run84_c0hex_$t.json').read().strip().splitlines()[-1]); print('scatter=$t', round(l['value'],3), round(l['roofline']['frac'],3))"; done
mkdir -p gpurun_out/r2run84
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:k_c0" -c 4 --csv --log-file gpurun_out/r2run84/launches.csv python bench.py --workload c0hex --steps 2 --warmup 1 --sweep off > /dev/null 2>&1
grep -E "k_c0" gpurun_out/r2run84/launches.csv | awk -F'","' '{print $(NF-2)" "$NF}' | head -6
