timeout 900 python -m pytest tests/test_assembly_gpu.py tests/test_multirank_gpu.py -m gpu -q > gpurun_out/r2run11_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2run11_pytest.log; grep -E "FAILED|Error" gpurun_out/r2run11_pytest.log | head
timeout 900 python bench.py --workload c0tet --sweep off > gpurun_out/r2run11_c0tet.json 2> gpurun_out/r2run11_c0tet.err; echo "c0tet rc=$?"
tail -c 600 gpurun_out/r2run11_c0tet.err
cut -c 1-600 gpurun_out/r2run11_c0tet.json
SK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --workload c0tet --elements 24000 --steps 3 --warmup 3 > gpurun_out/r2run11_c0tet_share2.json 2> gpurun_out/r2run11_c0tet_share2.err; echo "share rc=$?"
echo done
