# Full GPU suite + smoke + default bench line (+ reference arm when REF=1).
mkdir -p gpurun_out
T=${TAG:-r2x}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_gputests.log
tail -3 gpurun_out/${T}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
tail -2 gpurun_out/${T}_smoke.log
timeout 1700 python bench.py ${BENCH_ARGS} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${T}_bench.json')); print({k: d.get(k) for k in ('value','ttft_p99_ms','tbt_p99_ms','clocks')}, d['e2e']['value'], d['latency'].get('value'), d['latency'].get('ttft_p99_ms'), d['latency'].get('tbt_p99_ms'))
for k in d['kernels']: print(k['kernel'], k['frac'], k.get('frac_partition'), k['share_ms'])"
if [ -n "$REF" ]; then timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; tail -c 600 gpurun_out/${T}_ref.json; fi
