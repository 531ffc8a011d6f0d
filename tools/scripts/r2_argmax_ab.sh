# Sampling kernel change: kernel tests + engine token/logits parity, then pass timelines (argmax crit).
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "argmax or lm_head" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x 2>&1 | tail -2
for n in "3 2142 0" "48 1400 40" "78 1387 40"; do
  set -- $n
  python tools/timeline.py --n-dec $1 --ctx $2 --ppi-sms $3 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); c=d['classes'].get('argmax_emit_kernel',{})
print('n=$1', 'pass_ms', round(d['pass_ms_reported'],4), 'argmax', c)"
done
