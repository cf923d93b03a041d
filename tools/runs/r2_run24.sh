# ramped streamed chunk schedule: e2e A/B + streamed parity tests
timeout 600 python tools/e2e_chunks.py > gpurun_out/r2run24_e2e_chunks.jsonl 2> gpurun_out/r2run24.err; echo "rc=$?"
cat gpurun_out/r2run24_e2e_chunks.jsonl; tail -3 gpurun_out/r2run24.err
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "streamed" 2>&1 | tail -2
