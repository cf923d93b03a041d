# compute-sanitizer memcheck / racecheck / synccheck on the TMA pipelines and the default kernels (small sizes)
mkdir -p gpurun_out/r2run73
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "tma_paths and 17" > gpurun_out/r2run73/$tool.log 2>&1; echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/r2run73/$tool.log | tail -3
done
