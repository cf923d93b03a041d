# confirm the per-order M2 low-register table (op0) against all-off; parity on the new default
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_integration_speckern_gpu.py -m gpu -q -x > gpurun_out/r2run19_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run19_pytest.log
timeout 1200 python tools/tune_eb.py --variants op0,op0_lowreg0 --ops helm,stiff --orders 4-10 --gbytes 1.0 > gpurun_out/r2run19_lowreg.jsonl 2> gpurun_out/r2run19_lowreg.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run19_lowreg.err
echo done
