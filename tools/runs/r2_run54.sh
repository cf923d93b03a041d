# phys_deriv tile-width grid (own table and payload lane width) + pderiv parity on the main library
timeout 900 python -m pytest tests -m gpu -q -k "deriv or every_operator" > gpurun_out/r2run54_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run54_pytest.log; grep FAILED gpurun_out/r2run54_pytest.log | head
timeout 1800 python tools/tune_eb.py --variants op4,op4_eb16,op4_eb8,op4_eb4,op4_eb2,op4_eb1 --ops pderiv --orders 1-10 --gbytes 0.5 --reps 6 > gpurun_out/r2run54_pd.jsonl 2> gpurun_out/r2run54_pd.err; echo "tune rc=$?"
