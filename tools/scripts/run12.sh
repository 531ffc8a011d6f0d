timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k prefill 2>&1 | tail -2
timeout 600 python tools/kernel_probe.py --only chunk 2>&1 | tail -4
timeout 600 python tools/kernel_probe.py --only ppi 2>&1 | tail -4
CRONUS_PASS_STATS=1 timeout 300 python tools/one_pass.py --worker 1 --n-dec 32 --chunk 480 --pos0 2048 2>&1 | tail -2
