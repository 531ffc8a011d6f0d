# prefill kernel v3 (S double buffer): parity + probe + pipeline stamps
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "prefill or long_context" 2>&1 | tail -3
python tools/prefill_probe.py --ctas 108 --shapes 448x1024,448x0,448x3072,415x1024,200x0,1024x0,2048x0,64x1024,4096x0
python tools/prefill_probe.py --ctas -1 --shapes 448x1024,64x1024,4096x0
CRONUS_PF_PROBE=1 python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 1 2>&1 | tail -18
