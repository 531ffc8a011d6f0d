# ncu launch list (gpu__time_duration.sum) of a short bench command at the session-5 HEAD.
mkdir -p gpurun_out
CRONUS_NO_PDL=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/s5_ncu_launches_bench_final.csv python bench.py --requests 24 --warmup-requests 8 --warmup 1 --steps 1 \
  --no-cpu-baseline --no-e2e --no-profile --latency-load 0 --ppi-sms 0 > gpurun_out/s5_ncu_launch_final.log 2>&1
tail -1 gpurun_out/s5_ncu_launch_final.log | cut -c1-200; wc -l gpurun_out/s5_ncu_launches_bench_final.csv
