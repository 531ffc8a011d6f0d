# decode-attention ring depth chosen per launch (2 stages when the grid exceeds the 3-stage residency)
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q 2>&1 | tail -2
for r in 3 auto; do env $( [ $r = auto ] && echo X=1 || echo CRONUS_DEC_STAGES=$r ) timeout 300 python tools/pass_sweep.py llama3-8b 1x512 8x2048 16x2048 24x2048 32x2048 48x1024 64x2048 2>&1 | tail -1 | sed "s/^/dec_stages=$r /"; done
for r in 3 auto 3 auto; do env $( [ $r = auto ] && echo X=1 || echo CRONUS_DEC_STAGES=$r ) timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b28.json 2> gpurun_out/b28.err
python -c "
import json; d=json.load(open('gpurun_out/b28.json')); print('dec_stages=$r', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'))"; done
