# Measurement breadth on one B200 (BASELINE.json configs 3-5 at N=1, co-located pair):
#  * Qwen2-7B: calibrate, max req/s (all at t=0), fixed-interval sweep f in {0.5,0.7,0.9,1.0} of R_max
#  * LLaMA3-8B: the same interval sweep
#  * LLaMA3-8B long trace (4x paper means), 64 requests
set -u
B="python bench.py --no-cpu-baseline --no-e2e --no-profile --warmup 3"
timeout 600 python -m paper_2509_17357_b200.calibrate --model qwen2-7b --ppi-sms 40 --out gpurun_out/cfg_qwen.cfg > gpurun_out/calib_qwen.log 2>&1
for m in qwen2-7b llama3-8b; do
  cfg=tests/golden/configs/b200_llama8b_coloc.cfg; [ $m = qwen2-7b ] && cfg=gpurun_out/cfg_qwen.cfg
  timeout 900 $B --model $m --config $cfg > gpurun_out/sweep_${m}_max.json 2>gpurun_out/sweep_${m}_max.err
  R=$(python -c "import json; print(json.load(open('gpurun_out/sweep_${m}_max.json'))['value'])")
  for f in 0.5 0.7 0.9 1.0; do
    iv=$(python -c "print(1000.0/($f*$R))")
    timeout 900 $B --model $m --config $cfg --arrival fixed-interval --interval-ms $iv > gpurun_out/sweep_${m}_f$f.json 2>gpurun_out/sweep_${m}_f$f.err
  done
done
timeout 1200 $B --requests 64 --mean-in 4056 --mean-out 988 > gpurun_out/sweep_long.json 2>gpurun_out/sweep_long.err
for f in gpurun_out/sweep_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'], d['config']['trace'])" 2>/dev/null || echo "$f failed"; done
