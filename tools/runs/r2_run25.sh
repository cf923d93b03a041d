# PCIe pipeline probe (copies only / with a streaming kernel)
timeout 600 python tools/pcie_pipeline.py > gpurun_out/r2run25_pcie.jsonl 2> gpurun_out/r2run25.err; echo "rc=$?"
cat gpurun_out/r2run25_pcie.jsonl; tail -3 gpurun_out/r2run25.err
