# Recalibrate the co-located operating point for several SM splits and bench each.
for sms in 32 40 48; do
  timeout 600 python -m paper_2509_17357_b200.calibrate --ppi-sms $sms --out gpurun_out/cfg_$sms.cfg --samples-out gpurun_out/calib_$sms.json > gpurun_out/calib_$sms.log 2>&1
  timeout 900 python bench.py --ppi-sms $sms --config gpurun_out/cfg_$sms.cfg --no-cpu-baseline --no-e2e --no-profile > gpurun_out/bench_sms$sms.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_sms$sms.json')); print($sms, d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'], d['cpi_busy_ms'], d['cpi_lent_iterations'], d['cpi_iterations'])"
  grep "fit" gpurun_out/cfg_$sms.cfg | head -1
done
