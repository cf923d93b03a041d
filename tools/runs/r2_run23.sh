# e2e vs streamed chunk count (tet P=4, 2^20 elements)
timeout 600 python tools/e2e_chunks.py > gpurun_out/r2run23_e2e_chunks.jsonl 2> gpurun_out/r2run23.err; echo "rc=$?"
cat gpurun_out/r2run23_e2e_chunks.jsonl; tail -3 gpurun_out/r2run23.err
