# C0 hex fused gather with the element decomposition hoisted: assembly tests + c0hex bench
timeout 900 python -m pytest tests -m gpu -q -k "c0 or C0 or assembl or multirank" > gpurun_out/r2run83_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run83_pytest.log; grep FAILED gpurun_out/r2run83_pytest.log | head
for t in 1 2; do timeout 900 python bench.py --workload c0hex --sweep off > gpurun_out/r2run83_c0hex_$t.json 2>/dev/null; python3 -c "
import json; l=json.loads(open('gpurun_out/r2run83_c0hex_$t.json').read().strip().splitlines()[-1]); print('c0hex', round(l['value'],3), round(l['roofline']['frac'],3), round(l['e2e']['value'],3))"; done
