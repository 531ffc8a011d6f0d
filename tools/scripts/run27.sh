# decode attention TMA ring depth per warp on decode passes
for r in 3 2 4 6 3; do CRONUS_DEC_STAGES=$r timeout 300 python tools/pass_sweep.py llama3-8b 1x512 8x2048 16x2048 32x2048 64x2048 2>&1 | tail -1 | sed "s/^/dec_stages=$r /"; done
