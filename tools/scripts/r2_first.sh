mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_smoke.log
timeout 1700 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?" >> gpurun_out/r2a_bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err; echo "ref rc=$?" >> gpurun_out/r2a_ref.err
tail -3 gpurun_out/r2a_gputests.log; cat gpurun_out/r2a_bench.json | head -c 3000; cat gpurun_out/r2a_ref.json
