# even-odd mass sweeps at hex P=5: full GPU suite + mass A/B (op1 = new default vs the main-library mass table)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run42_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run42_pytest.log; grep FAILED gpurun_out/r2run42_pytest.log | head
SK_MASS_DENSE=0 timeout 900 python tools/tune_eb.py --variants op1 --ops mass --shapes hex --orders 4-6 --gbytes 1.0 > gpurun_out/r2run42_eo.jsonl 2> gpurun_out/r2run42_eo.err; echo "tune rc=$?"
cat gpurun_out/r2run42_eo.jsonl | cut -c 1-200 | head -3
