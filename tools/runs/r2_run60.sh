# zero-copy probe (kernel reads / writes pinned host memory over PCIe) vs the streamed apply
timeout 600 python tools/zero_copy_probe.py > gpurun_out/r2run60_zc.jsonl 2> gpurun_out/r2run60_zc.err; echo "rc=$?"
cat gpurun_out/r2run60_zc.jsonl; tail -3 gpurun_out/r2run60_zc.err
