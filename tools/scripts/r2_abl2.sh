# Split ablation with repeats: round-1 config vs the round-2 calibration (balancer), and fixed fractions;
# all-at-zero max throughput + fixed-interval latency at a common 14 req/s offered load.
python tools/gemm_probe.py 512 108 2>&1 | grep -E "probe|us"
Q="--no-cpu-baseline --no-e2e --no-profile --latency-load 0 --warmup 1"
A=tests/golden/configs/b200_llama8b_coloc.cfg
B=tests/golden/configs/b200_llama8b_coloc_r2fit.cfg
for rep in 1 2; do
for c in A B; do cfg=${!c}
  timeout 600 python bench.py $Q --config $cfg > gpurun_out/abl_${c}_$rep.json 2>/dev/null
  timeout 600 python bench.py $Q --config $cfg --arrival fixed-interval --interval-ms 71.43 > gpurun_out/abl_${c}_fi_$rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abl_${c}_$rep.json')); f=json.load(open('gpurun_out/abl_${c}_fi_$rep.json'))
print('$c rep$rep max', d['value'], 'fi14', f['value'], f['ttft_p99_ms'], f['tbt_p99_ms'], f['ttft_mean_ms'])"
done
CRONUS_FIXED_SPLIT=0.25 timeout 600 python bench.py $Q --config $B > gpurun_out/abl_F25_$rep.json 2>/dev/null
CRONUS_FIXED_SPLIT=0.25 timeout 600 python bench.py $Q --config $B --arrival fixed-interval --interval-ms 71.43 > gpurun_out/abl_F25_fi_$rep.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/abl_F25_$rep.json')); f=json.load(open('gpurun_out/abl_F25_fi_$rep.json'))
print('F25 rep$rep max', d['value'], 'fi14', f['value'], f['ttft_p99_ms'], f['tbt_p99_ms'], f['ttft_mean_ms'])"
done
