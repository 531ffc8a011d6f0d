timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "prefill or long_context" 2>&1 | tail -2
python tools/prefill_probe.py --ctas 108 --shapes 448x1024,448x0,448x3072,415x1024,200x0,1024x0,2048x0,64x1024,4096x0
python tools/prefill_probe.py --ctas 40 --shapes 200x0,512x0,1024x0,2048x0
