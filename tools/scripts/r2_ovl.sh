timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_engine_gpu.py -q -x 2>&1 | tail -2
for f in 0 0.25 0.35 0.5 0.7; do
  CRONUS_ATTN_OVERLAP=$f timeout 300 python tools/timeline.py --n-dec 80 --ctx 1440 --chunk 415 --pos0 1024 > /tmp/tl.log 2>&1
  python - <<PY
import json
t=open('/tmp/tl.log').read(); d=json.loads(t[t.index('{'):])
print('overlap=$f mixed 80x1440+415@1024 pass_ms', round(d['pass_ms_reported'],3))
PY
done
for n in 3 16; do timeout 300 python tools/timeline.py --n-dec $n --ctx 1400 > /tmp/tl.log 2>&1; python -c "
import json; t=open('/tmp/tl.log').read(); d=json.loads(t[t.index('{'):]); print('dec$n', round(d['pass_ms_reported'],3))"; done
