# full GPU suite + smoke with the TMA-fed mass on; mass / stiffness tables
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run33_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run33_pytest.log; grep -E "FAILED" gpurun_out/r2run33_pytest.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2run33_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --sweep on --sweep-tables mass_deformed,stiff_deformed --steps 5 > gpurun_out/r2run33_sweep.json 2> gpurun_out/r2run33_sweep.err; echo "sweep rc=$?"
tail -c 300 gpurun_out/r2run33_sweep.err
