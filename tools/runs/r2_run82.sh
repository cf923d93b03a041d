# C0 hex: mode-major elemental output + one-DOF-per-thread scatter (coalesced along x) A/B; assembly tests
timeout 900 python -m pytest tests -m gpu -q -k "c0 or C0 or assembl or multirank" > gpurun_out/r2run82_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run82_pytest.log; grep FAILED gpurun_out/r2run82_pytest.log | head
for t in 0 1 0 1; do SK_C0_HEX_MODEMAJOR=$t timeout 900 python bench.py --workload c0hex --sweep off > gpurun_out/r2run82_c0hex_$t.json 2>/dev/null; python3 -c "
import json; l=json.loads(open('gpurun_out/r2run82_c0hex_$t.json').read().strip().splitlines()[-1]); print('modemajor=$t', round(l['value'],3), round(l['roofline']['frac'],3), round(l['e2e']['value'],3))"; done
mkdir -p gpurun_out/r2run82
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_c0|k_tile|k_persist" -c 12 --csv --log-file gpurun_out/r2run82/launches.csv python bench.py --workload c0hex --steps 2 --warmup 1 --sweep off > /dev/null 2>&1
grep -E "k_c0|k_tile" gpurun_out/r2run82/launches.csv | awk -F'","' '{print $5" "$NF}' | cut -c 1-80,200- | head -6
