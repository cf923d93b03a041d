timeout 900 python -m pytest tests/test_assembly_gpu.py tests/test_multirank_gpu.py -m gpu -q > gpurun_out/r2run12_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2run12_pytest.log; grep -E "FAILED|Error" gpurun_out/r2run12_pytest.log | head
for w in c0pyr c0tet c0prism c0hex; do timeout 900 python bench.py --workload $w --sweep off > gpurun_out/r2run12_$w.json 2> gpurun_out/r2run12_$w.err; echo "$w rc=$?"; tail -c 300 gpurun_out/r2run12_$w.err; done
SK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --workload c0pyr --elements 24000 --steps 3 --warmup 3 > gpurun_out/r2run12_c0pyr_share2.json 2> gpurun_out/r2run12_c0pyr_share2.err; echo "share rc=$?"
echo done
