# CUDA-graph replay of decode passes: parity, per-pass A/B, serve A/B
CRONUS_GRAPH_STATS=1 timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -x -q 2>&1 | grep -v "^$" | tail -25
for g in 0 1; do CRONUS_GRAPHS=$g timeout 300 python tools/pass_sweep.py llama3-8b 1x512 8x512 8x2048 32x2048 64x2048 2>&1 | tail -1; done
for g in 0 1 0 1; do CRONUS_GRAPHS=$g CRONUS_GRAPH_STATS=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b15_$g.json 2> gpurun_out/b15_$g.err
python -c "
import json; d=json.load(open('gpurun_out/b15_$g.json')); print('graphs=$g', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'))"; grep graphs gpurun_out/b15_$g.err | sort | uniq -c | tail -4; done
