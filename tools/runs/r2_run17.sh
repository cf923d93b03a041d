timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run17_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run17_pytest.log; grep -E "FAILED|^E " gpurun_out/r2run17_pytest.log | head -20
echo done
