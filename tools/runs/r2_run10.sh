timeout 900 python -m pytest tests/test_assembly_gpu.py tests/test_multirank_gpu.py -m gpu -q > gpurun_out/r2run10_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2run10_pytest.log; grep -E "FAILED|Error" gpurun_out/r2run10_pytest.log | head
timeout 900 python bench.py --workload c0prism --sweep off > gpurun_out/r2run10_c0prism.json 2> gpurun_out/r2run10_c0prism.err; echo "c0prism rc=$?"
tail -c 600 gpurun_out/r2run10_c0prism.err
cat gpurun_out/r2run10_c0prism.json | cut -c 1-700
echo done
