timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run15_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run15_pytest.log; grep -E "FAILED" gpurun_out/r2run15_pytest.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2run15_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2run15_ref.json 2> gpurun_out/r2run15_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2run15_bench.json 2> gpurun_out/r2run15_bench.err; echo "bench rc=$?"
cut -c 1-1500 gpurun_out/r2run15_bench.json
echo done
