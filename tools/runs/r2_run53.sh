# non-collocated Helmholtz tile widths: full GPU suite + NC sweep
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run53_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run53_pytest.log; grep FAILED gpurun_out/r2run53_pytest.log | head
timeout 900 python tools/sweep.py --ops helmnc --orders 1-10 --gbytes 1.0 --reps 8 > gpurun_out/r2run53_nc.jsonl 2> gpurun_out/r2run53_nc.err; echo "sweep rc=$?"
