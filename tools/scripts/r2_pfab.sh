# Prefill attention: parity tests first (short timeouts: a pipeline deadlock must not hang the
# box), then CUDA-event timing at serve shapes and the pipeline clocks of CTA 0.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "prefill or long_context" 2>&1 | tail -3
for r in 1 2; do timeout 120 python tools/prefill_probe.py --shapes 448x1024,448x3072,415x1024,2048x0,4096x0 2>&1 | tail -5; done
timeout 60 python tools/prefill_probe.py --ctas -1 --shapes 448x1024,4096x0 2>&1 | tail -2
CRONUS_PF_PROBE=1 timeout 60 python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 1 2>&1 | grep -A14 "pf probe" | tail -15
