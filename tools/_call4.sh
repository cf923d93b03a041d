export PYTHONUNBUFFERED=1
L=paper_2604_04644_b200
timeout 300 python tools/check_helm.py > gpurun_out/c4_check.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c4_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/c4_gputests.log
timeout 500 python tools/tune_eb.py --variants op0,op0_rg1 --ops helm --geo regular --orders 1-10 --gbytes 1.0 > gpurun_out/c4_tune_regular.jsonl 2>&1
