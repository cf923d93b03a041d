export PYTHONUNBUFFERED=1
timeout 300 python tools/check_helm.py > gpurun_out/c6_check.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c6_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/c6_gputests.log
timeout 1200 python tools/sweep.py --ops helm,stiff,mass --orders 1-10 --gbytes 1.5 > gpurun_out/c6_sweep.jsonl 2> gpurun_out/c6_sweep.err
timeout 600 python tools/sweep.py --ops helm --geo regular --orders 1-10 --gbytes 1.5 > gpurun_out/c6_sweep_regular.jsonl 2>> gpurun_out/c6_sweep.err
