timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2run3_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2run3_pytest.log; grep FAILED gpurun_out/r2run3_pytest.log | head
for d in 0 1; do
  SK_MASS_DENSE=$d timeout 600 python tools/sweep.py --ops mass --orders 1-4 --gbytes 1.2 --reps 20 > gpurun_out/r2run3_mass_def_d$d.jsonl 2>&1
  SK_MASS_DENSE=$d timeout 600 python tools/sweep.py --ops mass --orders 1-6 --geo regular --gbytes 0.4 --reps 20 > gpurun_out/r2run3_mass_reg_d$d.jsonl 2>&1
done
timeout 900 python tools/sweep.py --ops helm,helmstaged --orders 2-10 --gbytes 1.2 --reps 10 > gpurun_out/r2run3_staged.jsonl 2>&1
echo done
