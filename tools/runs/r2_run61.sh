# direct-output streamed applies: streamed parity tests, e2e schedule A/B, default bench
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "streamed" 2>&1 | tail -1
timeout 600 python tools/e2e_chunks.py > gpurun_out/r2run61_e2e.jsonl 2> gpurun_out/r2run61_e2e.err; echo "rc=$?"
cat gpurun_out/r2run61_e2e.jsonl; tail -2 gpurun_out/r2run61_e2e.err
timeout 900 python bench.py --sweep off > gpurun_out/r2run61_bench.json 2> gpurun_out/r2run61_bench.err; echo "bench rc=$?"
