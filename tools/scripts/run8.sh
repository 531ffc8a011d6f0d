timeout 300 python tools/timeline.py --n-dec 1 --ctx 1024 --ppi-sms 0 --json gpurun_out/tl_dec1_148.json > /dev/null 2>&1
timeout 300 python tools/timeline.py --n-dec 8 --ctx 2048 --ppi-sms 0 --json gpurun_out/tl_dec8_148.json > /dev/null 2>&1
ls gpurun_out/
