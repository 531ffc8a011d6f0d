# The paper's comparison (Table 3 shape) on one B200: every policy on the same co-located
# pair, trace and profiles. Writes gpurun_out/policy_<p>.json.
for p in cronus dp disagg-lh disagg-hl; do
  timeout 900 python bench.py --policy $p --no-cpu-baseline --no-e2e --no-profile > gpurun_out/policy_$p.json 2> gpurun_out/policy_$p.err
  python -c "
import json; d=json.load(open('gpurun_out/policy_$p.json')); print('$p', d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'], d['violations'])" || tail -3 gpurun_out/policy_$p.err
done
