set -x
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py -m gpu -x -q -k "chain or decode" 2>&1 | tail -3
timeout 300 python tools/decode_bench.py --impl tma 2>&1 | tail -8
for w in 1.0 2.0 3.0; do timeout 300 python tools/decode_bench.py --impl tma --waves $w --shapes 8x1024,32x1024,8x2560,64x1024 2>&1 | tail -4; done
for pf in 0 1 2; do CRONUS_GEMM_L2PF=$pf timeout 600 python tools/kernel_probe.py --only decode 2>&1 | tail -8; done
