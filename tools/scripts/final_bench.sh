# Round-end evidence: default bench line, then the ncu launch list of a short bench command.
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json')); print({k: d.get(k) for k in ('value','ttft_p99_ms','tbt_p99_ms','e2e','handoff','gpu_launches')}); print(d['roofline']); print(d['cpu_baseline'])"
CRONUS_NO_PDL=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/ncu_launches_bench.csv python bench.py --requests 24 --warmup-requests 8 --warmup 1 --steps 1 \
  --no-cpu-baseline --no-e2e --no-profile --ppi-sms 0 > gpurun_out/ncu_launch_bench.log 2>&1
tail -2 gpurun_out/ncu_launch_bench.log; wc -l gpurun_out/ncu_launches_bench.csv
