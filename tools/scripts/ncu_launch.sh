B="python bench.py --requests 24 --warmup-requests 8 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e --no-profile"
for v in "CRONUS_NO_PDL=1 CRONUS_DECODE_CPASYNC=1" "CRONUS_NO_PDL=1 X=1" ; do
  env $v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/ncu_lb.csv $B > gpurun_out/ncu_lb.log 2>&1
  echo "== $v: $(wc -l < gpurun_out/ncu_lb.csv) lines"; grep ERROR gpurun_out/ncu_lb.log | head -3; tail -1 gpurun_out/ncu_lb.csv | cut -c1-200
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ncu_lb0.csv $B --ppi-sms 0 > gpurun_out/ncu_lb0.log 2>&1
echo "== sms0: $(wc -l < gpurun_out/ncu_lb0.csv)"; grep ERROR gpurun_out/ncu_lb0.log | head -3; tail -1 gpurun_out/ncu_lb0.csv | cut -c1-200
