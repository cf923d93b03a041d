# non-collocated Helmholtz tile-width grid (own table, own payload lane width) + NC parity on the main library
timeout 900 python -m pytest tests -m gpu -q -k "noncoll or nc or every_operator or streamed" > gpurun_out/r2run51_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run51_pytest.log; grep FAILED gpurun_out/r2run51_pytest.log | head
timeout 1800 python tools/tune_eb.py --variants op6,op6_eb16,op6_eb8,op6_eb4,op6_eb2,op6_eb1 --ops helmnc --orders 1-10 --gbytes 0.5 --reps 6 > gpurun_out/r2run51_nc.jsonl 2> gpurun_out/r2run51_nc.err; echo "tune rc=$?"
tail -2 gpurun_out/r2run51_nc.err
