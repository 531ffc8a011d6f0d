# Round-2 evidence: ncu launch list of a serve vs CUDA-event class timings (roofline check),
# tensor GEMM throughput alone (raw), then the sanitizers.
mkdir -p gpurun_out
CRONUS_NO_PDL=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/roof_launches.csv python tools/roofline_check.py serve --requests 24 \
  --stats gpurun_out/roof_stats_ncu.json > gpurun_out/roof_ncu.log 2>&1
timeout 600 python tools/roofline_check.py serve --requests 24 --stats gpurun_out/roof_stats_events.json > gpurun_out/roof_ev.log 2>&1
python tools/roofline_check.py compare gpurun_out/roof_launches.csv gpurun_out/roof_stats_ncu.json gpurun_out/roof_stats_events.json > gpurun_out/r2_roofline_check.json 2> gpurun_out/roof_cmp.err
head -c 3000 gpurun_out/r2_roofline_check.json; tail -3 gpurun_out/roof_cmp.err
timeout 600 python tools/gemm_tflops.py --m 512,1024,4096 --ctas 108,40,0 --reps 10 > gpurun_out/r2_gemm_tflops.jsonl 2>&1
CRONUS_GEMM_PAIR=0 timeout 600 python tools/gemm_tflops.py --m 512,4096 --ctas 108,0 --reps 10 > gpurun_out/r2_gemm_tflops_single.jsonl 2>&1
grep layer gpurun_out/r2_gemm_tflops.jsonl
bash tools/scripts/r2_sanitize.sh
