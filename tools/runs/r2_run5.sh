timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "dense or regular" > gpurun_out/r2run5_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2run5_pytest.log; grep FAILED gpurun_out/r2run5_pytest.log | head
for d in 0 1; do
  SK_HELM_DENSE=$d timeout 600 python tools/sweep.py --ops helm,stiff --orders 1-6 --geo regular --gbytes 0.3 --reps 10 > gpurun_out/r2run5_helm_reg_d$d.jsonl 2>&1
  SK_MASS_DENSE=$d timeout 600 python tools/sweep.py --ops mass --orders 1-6 --geo regular --gbytes 0.3 --reps 10 > gpurun_out/r2run5_mass_reg_d$d.jsonl 2>&1
done
echo done
