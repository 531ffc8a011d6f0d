timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k decode 2>&1 | tail -3
timeout 300 python tools/decode_bench.py --impl tma 2>&1 | tail -9
for c in 1 2 4 8 16; do timeout 300 python tools/decode_bench.py --impl tma --cluster $c --shapes 1x1024,1x4096,8x1024,8x2560 2>&1 | tail -4; done
PPI_SMS=0 timeout 300 python tools/pass_sweep.py llama3-8b 1x1024 8x1024 16x2048 32x1024 64x1024 128x1024 2>&1 | tail -1
PPI_SMS=40 timeout 300 python tools/pass_sweep.py llama3-8b 1x1024 8x1024 16x2048 32x1024 64x1024 128x1024 2>&1 | tail -1
