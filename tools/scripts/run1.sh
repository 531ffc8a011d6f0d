set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for impl in cp_async tma; do timeout 300 python tools/decode_bench.py --impl $impl 2>&1 | tail -8; done
for st in 2 4 6; do CRONUS_DEC_STAGES=$st timeout 300 python tools/decode_bench.py --impl tma 2>&1 | tail -8; done
