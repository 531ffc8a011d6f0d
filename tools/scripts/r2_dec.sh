# GEMM/decode parity after the warp-converged issue change + small-batch decode pass timelines.
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py -q -x 2>&1 | tail -2
for n in 3 8 32 95; do timeout 300 python tools/timeline.py --n-dec $n --ctx 2048 --ppi-sms 0 > gpurun_out/r2h_tl_dec$n.log 2>&1; python - <<PY
import json
t=open('gpurun_out/r2h_tl_dec$n.log').read(); d=json.loads(t[t.index('{'):])
print('dec$n', d['pass_ms_reported'], {k: (v['n'], v['crit_us_per_launch']) for k,v in d['classes'].items()})
PY
done
python tools/decode_bench.py --trace-lens --shapes 3x0,8x0,32x0,97x0
