# One `ncu --set full` capture per kernel class of the bench (CRONUS_NO_PDL=1: ncu replay
# cannot coexist with PDL dependents). Outputs gpurun_out/ncu_<name>.ncu-rep.
export CRONUS_NO_PDL=1
N="ncu --set full --clock-control none --import-source on"
$N -k regex:gemm_tc_kernel -s 169 -c 4 -o gpurun_out/ncu_gemm_stream_dec8 -f python tools/one_pass.py --worker 1 --n-dec 8 --ctx 2048 > gpurun_out/ncu1.log 2>&1
$N -k regex:attn_decode_tma -s 42 -c 1 -o gpurun_out/ncu_decode_attn_dec8 -f python tools/one_pass.py --worker 1 --n-dec 8 --ctx 2048 > gpurun_out/ncu2.log 2>&1
$N -k regex:attn_decode_tma -s 42 -c 1 -o gpurun_out/ncu_decode_attn_dec64 -f python tools/one_pass.py --worker 1 --n-dec 64 --ctx 1024 > gpurun_out/ncu3.log 2>&1
$N -k regex:gemm_tc_kernel -s 169 -c 4 -o gpurun_out/ncu_gemm_tc_ppi1024 -f python tools/one_pass.py --worker 0 --n-dec 0 --chunk 1024 > gpurun_out/ncu4.log 2>&1
$N -k regex:attn_prefill_tc -s 42 -c 1 -o gpurun_out/ncu_prefill_attn_chunk -f python tools/one_pass.py --worker 1 --n-dec 32 --chunk 480 --pos0 2048 > gpurun_out/ncu5.log 2>&1
ls -la gpurun_out/*.ncu-rep
