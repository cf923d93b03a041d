# final checks after the C0 changes: memcheck on the assembly tests, full GPU suite, smoke
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_assembly_gpu.py -m gpu -q > gpurun_out/r2run81_memcheck_c0.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2run81_memcheck_c0.log | tail -2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run81_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run81_pytest.log; grep FAILED gpurun_out/r2run81_pytest.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2run81_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2run81_smoke.log
