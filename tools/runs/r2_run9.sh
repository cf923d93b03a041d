timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run9_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2run9_pytest.log; grep FAILED gpurun_out/r2run9_pytest.log | head
timeout 1200 python bench.py --sweep on --sweep-quick --sweep-gb 100 --sweep-tables helm_deformed --steps 5 > gpurun_out/r2run9_maxsweep.json 2> gpurun_out/r2run9_maxsweep.err; echo "maxsweep rc=$?"
tail -c 400 gpurun_out/r2run9_maxsweep.err
echo done
