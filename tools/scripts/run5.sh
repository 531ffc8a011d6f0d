timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -x -q 2>&1 | tail -2
CRONUS_GEMM_RING_KB=100 timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -x -q 2>&1 | tail -2
for kb in 0 110 96 64; do echo "ring $kb"; CRONUS_GEMM_RING_KB=$kb timeout 600 python tools/kernel_probe.py --only decode 2>&1 | tail -8; done
