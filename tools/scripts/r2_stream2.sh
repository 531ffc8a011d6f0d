# 2 CTAs/SM weight streaming by token-tile size, on the 108-SM partition and on all 148 SMs
for ppi in 40 0; do for n in 3 16 24 32 48; do for k in 1 2; do
  CRONUS_GEMM_SK_PER_SM=$k CRONUS_GEMM_RING_KB=100 timeout 300 python tools/timeline.py --n-dec $n --ctx 1400 --ppi-sms $ppi > /tmp/tl.log 2>&1
  python -c "
import json; t=open('/tmp/tl.log').read(); d=json.loads(t[t.index('{'):]); print('ppi_sms=$ppi n_dec=$n per_sm=$k', round(d['pass_ms_reported'],3))"
done; done; done
CRONUS_NO_PDL=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/roof_launches.csv python tools/roofline_check.py serve --requests 8 --max-out 16 \
  --stats gpurun_out/roof_stats_ncu.json > gpurun_out/roof_ncu.log 2>&1
timeout 600 python tools/roofline_check.py serve --requests 8 --max-out 16 --stats gpurun_out/roof_stats_events.json > gpurun_out/roof_ev.log 2>&1
python tools/roofline_check.py compare gpurun_out/roof_launches.csv gpurun_out/roof_stats_ncu.json gpurun_out/roof_stats_events.json > gpurun_out/r2_roofline_check.json 2> gpurun_out/roof_cmp.err
python -c "
import json; d=json.load(open('gpurun_out/r2_roofline_check.json'))
for c in d['classes']: print(c)"; tail -3 gpurun_out/roof_cmp.err; tail -3 gpurun_out/roof_ncu.log
