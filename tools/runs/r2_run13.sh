timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run13_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run13_pytest.log; grep -E "FAILED" gpurun_out/r2run13_pytest.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2run13_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/r2run13_smoke.log
echo done
