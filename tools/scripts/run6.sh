for sms in 40 0; do for mega in 0 1; do PPI_SMS=$sms CRONUS_MEGA=$mega timeout 300 python tools/pass_sweep.py llama3-8b 8x1024 32x1024 64x1024 2>&1 | tail -1; done; done
PPI_SMS=0 CRONUS_GEMM_RING_KB=96 timeout 300 python tools/pass_sweep.py llama3-8b 8x1024 32x1024 64x1024 2>&1 | tail -1
