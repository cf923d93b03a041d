# round-2 closing run: GPU suite, smoke, reference arm, default bench
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run96_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run96_pytest.log; grep FAILED gpurun_out/r2run96_pytest.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2run96_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2run96_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/r2run96_ref.json 2> gpurun_out/r2run96_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/r2run96_bench.json 2> gpurun_out/r2run96_bench.err; echo "bench rc=$?"
