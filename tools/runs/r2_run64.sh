# regular-geometry TMA driver: full GPU suite on the main library (table on at tet P=9, prism P=5) and with it forced on everywhere
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run64_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run64_pytest.log; grep FAILED gpurun_out/r2run64_pytest.log | head
SK200_LIB=paper_2604_04644_b200/libsk200_htmar1.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run64_forced.log 2>&1; echo "forced rc=$?"
tail -1 gpurun_out/r2run64_forced.log; grep FAILED gpurun_out/r2run64_forced.log | head
