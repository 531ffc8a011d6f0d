# Prefill attention A/B at serve shapes: production vs dev variants (env), then the parity tests.
S=448x1024,448x3072,2048x0,4096x0
for v in "X=1" "CRONUS_PF_NPOLY=0" "CRONUS_PF_NPOLY=2"; do
  echo "== $v"; env $v python tools/prefill_probe.py --shapes $S 2>&1 | tail -4
done
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "prefill or long_context" 2>&1 | tail -2
