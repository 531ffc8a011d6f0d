# tensor-regime QKV stream-K (wave-fill gated): parity + serve A/B
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q 2>&1 | tail -2
for g in 0 1 0 1; do CRONUS_QKV_STREAMK=$g timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b17_$g.json 2> gpurun_out/b17_$g.err
python -c "
import json; d=json.load(open('gpurun_out/b17_$g.json')); print('qkv_streamk=$g', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'), d['iteration_shapes_count_ms_rows_ctx'].get('chunk+65-128'))"; done
