# auto decode residency for the cluster planner (3 per SM from 64 sequence x kv-head pairs)
CRONUS_DEC_SLOTS_PER_SM=0 timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 2 0; do CRONUS_DEC_SLOTS_PER_SM=$r timeout 300 python tools/pass_sweep.py llama3-8b 1x512 4x2048 8x2048 12x2048 16x2048 24x2048 32x2048 2>&1 | tail -1 | sed "s/^/slots=$r /"; done
for r in 2 0 2 0; do CRONUS_DEC_SLOTS_PER_SM=$r timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b32.json 2> gpurun_out/b32.err
python -c "
import json; d=json.load(open('gpurun_out/b32.json')); print('slots=$r', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'))"; done
