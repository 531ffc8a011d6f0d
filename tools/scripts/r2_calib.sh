# B200 calibration in the balancer's regime, then split ablation: balancer L_p vs fixed fractions.
mkdir -p gpurun_out
timeout 1500 python -m paper_2509_17357_b200.calibrate --model llama3-8b --ppi-sms 40 \
  --base tests/golden/configs/a100_a10_llama8b.cfg --out gpurun_out/b200_llama8b_coloc.cfg \
  --samples-out gpurun_out/r2_calibration_samples.json > gpurun_out/r2_calibration.log 2>&1
grep -E "^# fits" gpurun_out/b200_llama8b_coloc.cfg
Q="--no-cpu-baseline --no-e2e --no-profile --latency-load 0 --warmup 1"
for cfg in tests/golden/configs/b200_llama8b_coloc.cfg gpurun_out/b200_llama8b_coloc.cfg; do
  timeout 900 python bench.py $Q --config $cfg > gpurun_out/r2_abl_bal_$(basename $(dirname $cfg)).json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/r2_abl_bal_$(basename $(dirname $cfg)).json')); print('$cfg balancer', d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'])"
done
for f in 0.25 0.5 0.75; do
  CRONUS_FIXED_SPLIT=$f timeout 900 python bench.py $Q --config gpurun_out/b200_llama8b_coloc.cfg > gpurun_out/r2_abl_fixed_$f.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r2_abl_fixed_$f.json')); print('fixed $f', d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'])"
done
