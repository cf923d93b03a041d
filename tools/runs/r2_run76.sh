# tiled C0 scatter: C0 tests + c0hex bench A/B + ncu launch list
timeout 900 python -m pytest tests -m gpu -q -k "c0 or C0 or assembly or multirank" > gpurun_out/r2run76_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run76_pytest.log
for t in 0 1 0 1; do SK_C0_SCATTER_TILED=$t timeout 900 python bench.py --workload c0hex --sweep off > gpurun_out/r2run76_c0hex_$t.json 2>/dev/null; python3 -c "
import json; l=json.loads(open('gpurun_out/r2run76_c0hex_$t.json').read().strip().splitlines()[-1]); print('tiled=$t', round(l['value'],3), round(l['roofline']['frac'],3), round(l['e2e']['value'],3))"; done
mkdir -p gpurun_out/r2run76
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2run76/launches.csv python bench.py --workload c0hex --steps 2 --warmup 1 --sweep off > /dev/null 2>&1
grep -i scatter gpurun_out/r2run76/launches.csv | head -3 | cut -c 1-300
