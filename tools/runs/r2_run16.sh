timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -k dense > gpurun_out/r2run16_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2run16_pytest.log
for i in 1 2; do timeout 600 python tools/sweep.py --ops mass --orders 1-3 --gbytes 1.2 --reps 20 > gpurun_out/r2run16_mass_def_$i.jsonl 2>&1; done
echo done
