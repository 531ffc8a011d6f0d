# fused residual-GEMM RMSNorm (CK_FUSE_RMSNORM): kernel + engine parity, pass sweep and serve A/B
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -x -q 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q 2>&1 | tail -3
for g in 0 16 64; do CRONUS_NORM_FUSE_ROWS=$g timeout 300 python tools/pass_sweep.py llama3-8b 1x512 8x2048 16x2048 32x2048 64x2048 2>&1 | tail -1 | sed "s/^/rows=$g /"; done
for g in 0 16 0 16; do CRONUS_NORM_FUSE_ROWS=$g timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b21_$g.json 2> gpurun_out/b21_$g.err
python -c "
import json; d=json.load(open('gpurun_out/b21_$g.json')); print('norm_fuse_rows=$g', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'))"; done
