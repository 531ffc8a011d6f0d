# hybrid whole-tile / stream-K-tail SiLU GEMM: kernel + engine parity, pass and serve A/B
timeout 600 python -m pytest tests/test_gemm_gpu.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q 2>&1 | tail -2
for g in 0 1; do CRONUS_SILU_HYBRID=$g timeout 300 python tools/timeline.py --n-dec 76 --ctx 1024 --chunk 436 --pos0 1024 > gpurun_out/tl19_$g.txt 2>&1; grep -m1 pass_ms gpurun_out/tl19_$g.txt; done
for g in 0 1 0 1 0 1; do CRONUS_SILU_HYBRID=$g timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b19_$g.json 2> gpurun_out/b19_$g.err
python -c "
import json; d=json.load(open('gpurun_out/b19_$g.json')); print('silu_hybrid=$g', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'), d['iteration_shapes_count_ms_rows_ctx'].get('chunk+65-128'))"; done
