# CTA-pair GEMM: parity (single vs pair) and throughput
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -3
for pr in 0 1; do echo "CRONUS_GEMM_PAIR=$pr"; CRONUS_GEMM_PAIR=$pr timeout 300 python tools/gemm_tflops.py --m 512,1024,4096 --ctas 108,40,0 --reps 10 2>&1 | grep layer; done
