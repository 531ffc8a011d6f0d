timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "prefill" 2>&1 | tail -15
