timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2run2_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2run2_pytest.log
for d in 0 1; do
  SK_MASS_DENSE=$d timeout 600 python tools/sweep.py --ops mass --orders 1-4 --gbytes 1.2 --reps 20 > gpurun_out/r2run2_mass_def_d$d.jsonl 2>&1
  SK_MASS_DENSE=$d timeout 600 python tools/sweep.py --ops mass --orders 1-4 --geo regular --gbytes 0.4 --reps 20 > gpurun_out/r2run2_mass_reg_d$d.jsonl 2>&1
done
echo done
