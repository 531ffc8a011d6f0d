# weight-streaming GEMM: bytes in flight per SM (ring size x CTAs per SM) on decode passes
for cfg in "100 1" "100 2" "0 1" "150 1" "60 2"; do set -- $cfg
  for n in 3 16 81; do
    CRONUS_GEMM_RING_KB=$1 CRONUS_GEMM_SK_PER_SM=$2 timeout 300 python tools/timeline.py --n-dec $n --ctx 1400 > /tmp/tl.log 2>&1
    python - <<PY
import json
t=open('/tmp/tl.log').read(); d=json.loads(t[t.index('{'):])
g=[v for k,v in d['classes'].items() if k.startswith('gemm')]
print('ring=$1 per_sm=$2 n_dec=$n pass_ms', round(d['pass_ms_reported'],3), 'gemm crit us/launch', [round(x['crit_us_per_launch'],2) for x in g])
PY
  done
done
# mixed-pass attention overlap (prefill attention on the side stream) at several CTA shares
for f in 0 0.25 0.35 0.5; do
  CRONUS_ATTN_OVERLAP=$f timeout 300 python tools/kernel_probe.py --only chunk --reps 5 2>&1 | sed "s/^/overlap=$f /"
  CRONUS_ATTN_OVERLAP=$f timeout 300 python tools/timeline.py --n-dec 80 --ctx 1440 --chunk 415 --pos0 1024 > /tmp/tl.log 2>&1
  python - <<PY
import json
t=open('/tmp/tl.log').read(); d=json.loads(t[t.index('{'):])
print('overlap=$f mixed 80x1440+415@1024 pass_ms', round(d['pass_ms_reported'],3))
PY
done
