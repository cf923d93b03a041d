# Helmholtz / stiffness GPU tests with the low-register metric sweep forced on everywhere
SK200_LIB=paper_2604_04644_b200/libsk200_lowreg1.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run40_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run40_pytest.log; grep FAILED gpurun_out/r2run40_pytest.log | head
