# bwd_trans tile widths: full GPU suite + bwd / staged sweep
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run50_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run50_pytest.log; grep FAILED gpurun_out/r2run50_pytest.log | head
timeout 900 python tools/sweep.py --ops bwd --orders 1-10 --gbytes 1.0 --reps 8 > gpurun_out/r2run50_bwd.jsonl 2> gpurun_out/r2run50_bwd.err; echo "sweep rc=$?"
