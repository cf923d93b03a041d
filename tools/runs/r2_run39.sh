# full GPU suite with the TMA drivers forced on for every (shape, order) (k_persist_tma for deformed Helmholtz / stiffness, k_mass_tma for deformed mass)
SK200_LIB=paper_2604_04644_b200/libsk200_htma1_mtma1.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run39_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/r2run39_pytest.log; grep FAILED gpurun_out/r2run39_pytest.log | head
