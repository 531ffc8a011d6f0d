# wave-count rule for the decode-attention ring depth
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 3 auto; do env $( [ $r = auto ] && echo X=1 || echo CRONUS_DEC_STAGES=$r ) timeout 300 python tools/pass_sweep.py llama3-8b 16x2048 24x2048 32x2048 48x1024 64x2048 76x1024 2>&1 | tail -1 | sed "s/^/dec_stages=$r /"; done
