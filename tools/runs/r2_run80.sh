# mapped C0 with the gather fused into the elemental kernel: assembly tests + bench A/B
timeout 900 python -m pytest tests -m gpu -q -k "c0 or C0 or assembl or multirank" > gpurun_out/r2run80_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run80_pytest.log; grep FAILED gpurun_out/r2run80_pytest.log | head
for w in c0prism c0tet c0pyr; do for t in 0 1; do SK_C0_FUSED=$t timeout 900 python bench.py --workload $w --sweep off > gpurun_out/r2run80_${w}_$t.json 2>/dev/null; python3 -c "
import json; l=json.loads(open('gpurun_out/r2run80_${w}_$t.json').read().strip().splitlines()[-1]); print('$w fused=$t', round(l['value'],3), round(l['roofline']['frac'],3), round(l['e2e']['value'],3))"; done; done
