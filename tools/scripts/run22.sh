# SiLU * up in the stream-K gate_up GEMM's tile finalize for decode passes (CRONUS_SILU_FUSE_ROWS)
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -x -q -k "fused_silu or rmsnorm" 2>&1 | tail -2
CRONUS_SILU_FUSE_ROWS=128 timeout 1500 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q 2>&1 | tail -2
for g in 0 16 128; do CRONUS_SILU_FUSE_ROWS=$g timeout 300 python tools/pass_sweep.py llama3-8b 1x512 8x2048 16x2048 32x2048 64x2048 2>&1 | tail -1 | sed "s/^/silu_rows=$g /"; done
for g in 0 128 0 128; do CRONUS_SILU_FUSE_ROWS=$g timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b22_$g.json 2> gpurun_out/b22_$g.err
python -c "
import json; d=json.load(open('gpurun_out/b22_$g.json')); print('silu_fuse_rows=$g', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'))"; done
