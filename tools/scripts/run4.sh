timeout 300 python tools/timeline.py --n-dec 8 --ctx 1024 --json gpurun_out/tl_dec8.json > gpurun_out/tl_dec8.txt 2>&1
timeout 300 python tools/timeline.py --n-dec 64 --ctx 1024 --json gpurun_out/tl_dec64.json > gpurun_out/tl_dec64.txt 2>&1
timeout 300 python tools/timeline.py --n-dec 32 --ctx 1024 --chunk 480 --json gpurun_out/tl_chunk.json > gpurun_out/tl_chunk.txt 2>&1
tail -30 gpurun_out/tl_dec8.txt
