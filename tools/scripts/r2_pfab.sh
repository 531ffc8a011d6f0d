# Prefill attention: parity tests first (short timeout: a pipeline deadlock must not hang the
# box), then CUDA-event timing at serve shapes with / without the exp ping-pong (ablate bit 6),
# and the pipeline clocks of CTA 0 (448 @ 1024, no split).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "prefill or long_context" 2>&1 | tail -3
for v in "X=1" "CRONUS_PF_ABLATE=64" "CRONUS_PF_NPOLY=1"; do
  echo "== $v"; env $v timeout 120 python tools/prefill_probe.py --shapes 448x1024,448x3072,415x1024,2048x0,4096x0 2>&1 | tail -5
done
timeout 60 python tools/prefill_probe.py --ctas 27 --shapes 415x1024 2>&1 | tail -1
CRONUS_PF_PROBE=1 timeout 60 python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 1 2>&1 | tail -18 | head -18
