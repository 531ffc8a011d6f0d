timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "prefill or long_context" 2>&1 | tail -2
for ab in 0 8; do echo "ablate=$ab"; CRONUS_PF_ABLATE=$ab python tools/prefill_probe.py --ctas 108 --shapes 448x1024,448x3072,2048x0,4096x0; done
CRONUS_PF_PROBE=1 python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 1 2>&1 | tail -18 | head -8
