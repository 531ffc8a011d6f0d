# Iteration check: kernel parity, kernel probes, one mixed-pass timeline, the default bench line.
mkdir -p gpurun_out
T=${TAG:-r2d}
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_decode_plan.py -q -x > gpurun_out/${T}_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_kernels.log
tail -3 gpurun_out/${T}_kernels.log
timeout 300 python tools/prefill_probe.py --ctas 108 --shapes 448x1024,448x0,448x3072,415x1024,200x0,1024x0,2048x0,64x1024,4096x0 > gpurun_out/${T}_prefill_probe108.log 2>&1
timeout 300 python tools/prefill_probe.py --ctas 40 --shapes 200x0,512x0,1024x0,2048x0 > gpurun_out/${T}_prefill_probe40.log 2>&1
timeout 300 python tools/prefill_probe.py --ctas -1 --shapes 448x1024,200x0,4096x0 > gpurun_out/${T}_prefill_probe_nosplit.log 2>&1
cat gpurun_out/${T}_prefill_probe*.log
for pl in engine r1; do timeout 300 python tools/decode_bench.py --trace-lens --planner $pl --shapes 97x0,32x0,8x0,128x0 >> gpurun_out/${T}_decode_trace.log 2>&1; done
cat gpurun_out/${T}_decode_trace.log
timeout 300 python tools/timeline.py --n-dec 97 --ctx 1395 --chunk 415 --pos0 1024 > gpurun_out/${T}_tl_mixed.log 2>&1
if [ -z "$NOBENCH" ]; then
timeout 1700 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${T}_bench.json')); print({k: d.get(k) for k in ('value','ttft_p99_ms','tbt_p99_ms')}, d['e2e']['value'], d['latency'].get('value'))
for k in d['kernels']: print(k['kernel'], k['frac'], k.get('frac_partition'), k['share_ms'])"
fi
