# phys_deriv tile widths: full GPU suite + sweep of every other operator
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run55_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run55_pytest.log; grep FAILED gpurun_out/r2run55_pytest.log | head
timeout 1500 python tools/sweep.py --ops bwd,iprod,pderiv,ipderiv,helmnc --orders 1-10 --gbytes 1.0 --reps 8 > gpurun_out/r2run55_ops.jsonl 2> gpurun_out/r2run55_ops.err; echo "sweep rc=$?"
