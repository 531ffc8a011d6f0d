mkdir -p gpurun_out
CRONUS_NO_PDL=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/roof_launches.csv python tools/roofline_check.py serve --requests 24 \
  --stats gpurun_out/roof_stats_ncu.json > gpurun_out/roof_ncu.log 2>&1
timeout 600 python tools/roofline_check.py serve --requests 24 --stats gpurun_out/roof_stats_events.json > gpurun_out/roof_ev.log 2>&1
python tools/roofline_check.py compare gpurun_out/roof_launches.csv gpurun_out/roof_stats_ncu.json gpurun_out/roof_stats_events.json > gpurun_out/r2_roofline_check.json 2> gpurun_out/roof_cmp.err
cat gpurun_out/r2_roofline_check.json | python -c "
import json,sys; d=json.load(sys.stdin)
for c in d['classes']: print(c)"; tail -3 gpurun_out/roof_cmp.err; tail -3 gpurun_out/roof_ncu.log
