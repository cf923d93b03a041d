# confirm the kHelmTma table (op0) against all-off; full GPU suite on the main library
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run37_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run37_pytest.log; grep FAILED gpurun_out/r2run37_pytest.log | head
timeout 1500 python tools/tune_eb.py --variants op0,op0_htma0,op0 --ops helm,stiff --orders 2-10 --gbytes 1.0 > gpurun_out/r2run37_htma.jsonl 2> gpurun_out/r2run37_htma.err; echo "tune rc=$?"
