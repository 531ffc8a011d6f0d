# Weight-streaming gate_up: stream-K + SiLU kernel (default) vs hybrid whole-tile SiLU epilogue.
mkdir -p gpurun_out
CRONUS_SILU_HYBRID_ROWS=1 timeout 900 python -m pytest tests/test_engine_8b_gpu.py tests/test_engine_gpu.py -q -x 2>&1 | tail -2
for n in 17 43 78 128; do
  for v in "X=1" "CRONUS_SILU_HYBRID_ROWS=1"; do
    r=$(env $v python tools/timeline.py --n-dec $n --ctx 1387 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['pass_ms_reported'],4), d['kernels'])")
    echo "n=$n 108 SMs [$v] pass_ms kernels: $r"
  done
done
for n in 43 78; do
  for v in "X=1" "CRONUS_SILU_HYBRID_ROWS=1"; do
    r=$(env $v python tools/timeline.py --n-dec $n --ctx 1387 --ppi-sms 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['pass_ms_reported'],4), d['kernels'])")
    echo "n=$n 148 SMs [$v] pass_ms kernels: $r"
  done
done
