timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
PPI_SMS=0 timeout 300 python tools/pass_sweep.py llama3-8b 1x1024 8x1024 16x2048 32x1024 64x1024 128x1024 2>&1 | tail -1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'])"
