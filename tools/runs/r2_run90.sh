timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run90_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run90_pytest.log; grep FAILED gpurun_out/r2run90_pytest.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for w in c0hex; do timeout 900 python bench.py --workload $w --sweep off 2>/dev/null | python3 -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', round(l['value'],3))"; done
