# weight-stream GEMM ring size (BN <= 32 stream-K) on decode passes, graphs on (default)
for r in 100 64 140 0 100; do CRONUS_GEMM_RING_KB=$r timeout 300 python tools/pass_sweep.py llama3-8b 1x512 4x2048 8x2048 16x2048 32x2048 2>&1 | tail -1 | sed "s/^/ring_kb=$r /"; done
