# Round-2 diagnostics: logits tolerance stats, full GPU suite, per-pass timelines, kernel probes.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_8b_gpu.py -k logits -q -s > gpurun_out/r2b_logits.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2b_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b_gputests.log
timeout 300 python tools/timeline.py --n-dec 97 --ctx 1395 --chunk 415 --pos0 1024 > gpurun_out/r2b_tl_mixed.log 2>&1
timeout 300 python tools/timeline.py --n-dec 3 --ctx 2181 > gpurun_out/r2b_tl_dec3.log 2>&1
timeout 300 python tools/timeline.py --n-dec 95 --ctx 1429 > gpurun_out/r2b_tl_dec95.log 2>&1
timeout 300 python tools/prefill_probe.py > gpurun_out/r2b_prefill_probe.log 2>&1
timeout 300 python tools/decode_bench.py --shapes 3x2181,32x1792,96x1400,64x1024,128x1024 > gpurun_out/r2b_decode_bench.log 2>&1
tail -3 gpurun_out/r2b_gputests.log; grep "max |d" gpurun_out/r2b_logits.log; cat gpurun_out/r2b_prefill_probe.log gpurun_out/r2b_decode_bench.log
