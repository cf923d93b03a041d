timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "tma_paths" 2>&1 | tail -2
