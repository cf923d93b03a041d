# full GPU suite + default bench (with the helm_recompute table and the e2e copy ceiling)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run22_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run22_pytest.log; grep -E "FAILED" gpurun_out/r2run22_pytest.log | head
timeout 900 python bench.py > gpurun_out/r2run22_bench.json 2> gpurun_out/r2run22_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2run22_bench.err
echo done
