# Round-2 final evidence: Qwen2-7B calibration, ncu --set full of the production kernels at the
# C2 serve's shapes, the ncu launch list of a short bench command.
mkdir -p gpurun_out
timeout 1500 python -m paper_2509_17357_b200.calibrate --model qwen2-7b --ppi-sms 40 \
  --base tests/golden/configs/a100_a30_qwen7b.cfg --out gpurun_out/b200_qwen7b_coloc.cfg \
  --samples-out gpurun_out/r2_calibration_samples_qwen.json > gpurun_out/r2_calibration_qwen.log 2>&1
grep "^# fits" gpurun_out/b200_qwen7b_coloc.cfg
export CRONUS_NO_PDL=1
N="timeout 600 ncu --set full --clock-control none --import-source on"
M="--worker 1 --n-dec 80 --ctx 1440 --chunk 415 --pos0 1024"
$N -k regex:attn_prefill_pp -s 40 -c 1 -o gpurun_out/ncu2_prefill_pp_mixed -f python tools/one_pass.py $M > gpurun_out/ncu2_a.log 2>&1
$N -k regex:attn_decode_tma -s 40 -c 1 -o gpurun_out/ncu2_decode_mixed -f python tools/one_pass.py $M > gpurun_out/ncu2_b.log 2>&1
$N -k regex:gemm_tc_kernel -s 161 -c 4 -o gpurun_out/ncu2_gemm_tc_mixed -f python tools/one_pass.py $M > gpurun_out/ncu2_c.log 2>&1
$N -k regex:gemm_tc_kernel -s 161 -c 4 -o gpurun_out/ncu2_gemm_stream_dec8 -f python tools/one_pass.py --worker 1 --n-dec 8 --ctx 2048 > gpurun_out/ncu2_d.log 2>&1
$N -k regex:attn_prefill_pp -s 40 -c 1 -o gpurun_out/ncu2_prefill_pp_ppi -f python tools/one_pass.py --worker 0 --n-dec 0 --chunk 512 > gpurun_out/ncu2_e.log 2>&1
ls -la gpurun_out/ncu2_*.ncu-rep
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/ncu2_launches_bench.csv python bench.py --requests 24 --warmup-requests 8 --warmup 1 --steps 1 \
  --no-cpu-baseline --no-e2e --no-profile --latency-load 0 --ppi-sms 0 > gpurun_out/ncu2_launch_bench.log 2>&1
tail -2 gpurun_out/ncu2_launch_bench.log; wc -l gpurun_out/ncu2_launches_bench.csv
CRONUS_NO_PDL=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/roof_launches.csv python tools/roofline_check.py serve --requests 8 --max-out 16 --no-warm \
  --stats gpurun_out/roof_stats_ncu.json > gpurun_out/roof_ncu.log 2>&1
timeout 600 python tools/roofline_check.py serve --requests 8 --max-out 16 --no-warm --stats gpurun_out/roof_stats_events.json > gpurun_out/roof_ev.log 2>&1
python tools/roofline_check.py compare gpurun_out/roof_launches.csv gpurun_out/roof_stats_ncu.json gpurun_out/roof_stats_events.json > gpurun_out/r2_roofline_check.json 2> gpurun_out/roof_cmp.err
python -c "
import json; d=json.load(open('gpurun_out/r2_roofline_check.json'))
for c in d['classes']: print(c)"
