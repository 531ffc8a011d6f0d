# Calibration in the balancer's regime + ncu --set full of the production kernels at serve shapes.
mkdir -p gpurun_out
timeout 1200 python -m paper_2509_17357_b200.calibrate --model llama3-8b --ppi-sms 40 \
  --base tests/golden/configs/a100_a10_llama8b.cfg --out gpurun_out/b200_llama8b_coloc.cfg \
  --samples-out gpurun_out/r2_calibration_samples.json > gpurun_out/r2_calibration.log 2>&1
export CRONUS_NO_PDL=1
N="timeout 600 ncu --set full --clock-control none --import-source on"
# mixed pass of the C2 serve (97 decoders x 1395 keys + a 415-token chunk at 1024)
$N -k regex:attn_prefill_pp -s 40 -c 1 -o gpurun_out/ncu_prefill_pp_mixed -f python tools/one_pass.py --worker 1 --n-dec 97 --ctx 1395 --chunk 415 --pos0 1024 > gpurun_out/ncu_a.log 2>&1
$N -k regex:attn_decode_tma -s 40 -c 1 -o gpurun_out/ncu_decode_mixed -f python tools/one_pass.py --worker 1 --n-dec 97 --ctx 1395 --chunk 415 --pos0 1024 > gpurun_out/ncu_b.log 2>&1
$N -k regex:gemm_tc_kernel -s 161 -c 4 -o gpurun_out/ncu_gemm_tc_mixed -f python tools/one_pass.py --worker 1 --n-dec 97 --ctx 1395 --chunk 415 --pos0 1024 > gpurun_out/ncu_c.log 2>&1
$N -k regex:gemm_tc_kernel -s 161 -c 4 -o gpurun_out/ncu_gemm_stream_dec8 -f python tools/one_pass.py --worker 1 --n-dec 8 --ctx 2048 > gpurun_out/ncu_d.log 2>&1
$N -k regex:attn_prefill_pp -s 40 -c 1 -o gpurun_out/ncu_prefill_pp_ppi -f python tools/one_pass.py --worker 0 --n-dec 0 --chunk 512 > gpurun_out/ncu_e.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -30 gpurun_out/r2_calibration.log
