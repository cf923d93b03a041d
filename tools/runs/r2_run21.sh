# recomputed-metric Helmholtz: parity tests, then the helm_recompute + helm_deformed tables (all orders)
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "recomputed" > gpurun_out/r2run21_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run21_pytest.log; grep -E "Error|assert" gpurun_out/r2run21_pytest.log | head -5
timeout 1200 python bench.py --sweep on --sweep-tables helm_recompute,helm_deformed --steps 5 > gpurun_out/r2run21_sweep.json 2> gpurun_out/r2run21_sweep.err; echo "sweep rc=$?"
tail -c 600 gpurun_out/r2run21_sweep.err
echo done
