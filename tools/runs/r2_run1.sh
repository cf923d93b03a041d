timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2run1_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2run1_pytest.log
timeout 600 python bench.py > gpurun_out/r2run1_bench.json 2> gpurun_out/r2run1_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --workload hex4 --sweep off > gpurun_out/r2run1_hex4.json 2> gpurun_out/r2run1_hex4.err; echo "hex4 rc=$?"
timeout 300 python bench.py --workload mixed6 > gpurun_out/r2run1_mixed6.json 2> gpurun_out/r2run1_mixed6.err; echo "mixed6 rc=$?"
tail -c 600 gpurun_out/r2run1_bench.err
