# Session-5 round-end evidence: GPU suite + smoke + default bench + reference arm, the ncu launch
# list of a short bench command, ncu --set full of the production prefill kernel (448 @ 1024) and
# of the decode attention at tail shapes (planner choice), decode planner sweep.
mkdir -p gpurun_out
REF=1 TAG=r2s9 bash tools/scripts/r2_full.sh
export CRONUS_NO_PDL=1
N="timeout 600 ncu --set full --clock-control none --import-source on"
$N -k regex:attn_prefill_pp -s 5 -c 1 -o gpurun_out/s5_ncu_prefill_448x1024 -f python tools/prefill_probe.py --shapes 448x1024 --reps 1 > gpurun_out/s5_ncu_a.log 2>&1
$N -k regex:attn_decode_tma -s 5 -c 1 -o gpurun_out/s5_ncu_decode_1x2142 -f python tools/decode_bench.py --shapes 1x2142 --reps 1 > gpurun_out/s5_ncu_b.log 2>&1
$N -k regex:attn_decode_tma -s 5 -c 1 -o gpurun_out/s5_ncu_decode_16x2048 -f python tools/decode_bench.py --shapes 16x2048 --reps 1 > gpurun_out/s5_ncu_c.log 2>&1
unset CRONUS_NO_PDL
CRONUS_NO_PDL=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/s5_ncu_launches_bench.csv python bench.py --requests 24 --warmup-requests 8 --warmup 1 --steps 1 \
  --no-cpu-baseline --no-e2e --no-profile --latency-load 0 --ppi-sms 0 > gpurun_out/s5_ncu_launch_bench.log 2>&1
tail -2 gpurun_out/s5_ncu_launch_bench.log; wc -l gpurun_out/s5_ncu_launches_bench.csv
ls -la gpurun_out/*.ncu-rep
