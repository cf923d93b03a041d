set -x
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown --format=csv -lms 200 > gpurun_out/r2base_smi.csv &
SMI=$!
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2base_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2base_pytest.log
timeout 900 python tools/sweep.py --ops helm,stiff,mass --orders 2-10 --gbytes 1.5 --reps 20 > gpurun_out/r2base_sweep.jsonl 2> gpurun_out/r2base_sweep.err; echo "sweep rc=$?"
kill $SMI
