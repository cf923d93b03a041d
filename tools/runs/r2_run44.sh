# mass even-odd table: full GPU suite + mass table
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run44_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run44_pytest.log; grep FAILED gpurun_out/r2run44_pytest.log | head
timeout 1200 python bench.py --sweep on --sweep-tables mass_deformed --steps 5 > gpurun_out/r2run44_sweep.json 2> gpurun_out/r2run44_sweep.err; echo "sweep rc=$?"
