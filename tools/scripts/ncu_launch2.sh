# ncu launch list of a whole short serve (24 requests, no warm-up: the timed serve is all of it) next to the
# CUPTI critical-path shares bench.py computes for the same serve. --ppi-sms 0: ncu cannot prepare kernels
# launched into green-context streams in this mode.
B="python bench.py --requests 24 --warmup 0 --steps 1 --ppi-sms 0 --no-cpu-baseline --no-e2e"
CRONUS_NO_PDL=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file gpurun_out/ncu_launches_serve24.csv $B --no-profile > gpurun_out/ncu_ls.log 2>&1
echo "lines $(wc -l < gpurun_out/ncu_launches_serve24.csv)"; grep ERROR gpurun_out/ncu_ls.log | head -2
timeout 900 $B --profile-requests 24 > gpurun_out/bench_serve24.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_serve24.json')); print(d['value']); [print(k['kernel'], k['share_ms'], k['launches']) for k in d['kernels']]"
