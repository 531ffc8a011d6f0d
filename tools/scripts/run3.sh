set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/kernel_probe.py 2>&1 | tail -20
