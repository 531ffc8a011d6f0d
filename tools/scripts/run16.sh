timeout 300 python tools/timeline.py --n-dec 76 --ctx 1024 --chunk 436 --pos0 1024 > gpurun_out/tl_mixed.txt 2>&1
timeout 300 python tools/timeline.py --n-dec 0 --ctx 1024 --chunk 436 --pos0 1024 > gpurun_out/tl_chunk.txt 2>&1
timeout 300 python tools/timeline.py --n-dec 76 --ctx 1024 --chunk 0 --pos0 0 > gpurun_out/tl_dec76.txt 2>&1
