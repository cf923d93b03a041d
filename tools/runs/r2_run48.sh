# per-operator launch overrides: full GPU suite + the other operators' sweep
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run48_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run48_pytest.log; grep FAILED gpurun_out/r2run48_pytest.log | head
timeout 1500 python tools/sweep.py --ops bwd,iprod,pderiv,ipderiv,helmnc --orders 1-10 --gbytes 1.0 --reps 8 > gpurun_out/r2run48_ops.jsonl 2> gpurun_out/r2run48_ops.err; echo "sweep rc=$?"
