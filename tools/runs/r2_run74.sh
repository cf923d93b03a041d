# compute-sanitizer memcheck over the whole parity suite; racecheck over the TMA / dense / streamed tests
mkdir -p gpurun_out/r2run74
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_parity_gpu.py -m gpu -q > gpurun_out/r2run74/memcheck.log 2>&1; echo "memcheck rc=$?"
grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2run74/memcheck.log | tail -3
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "tma_paths or dense_dmma_mass or recomputed or staged" > gpurun_out/r2run74/racecheck.log 2>&1; echo "racecheck rc=$?"
grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/r2run74/racecheck.log | tail -3
