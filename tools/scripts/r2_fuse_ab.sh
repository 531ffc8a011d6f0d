# Small decode passes (148 SMs, the all-at-t=0 tail): pass time with the RMSNorm / SiLU fused into
# the GEMM tile finalizes vs separate kernels.
mkdir -p gpurun_out
for n in 1 3 8; do
  for v in "X=1" "CRONUS_NORM_FUSE_ROWS=16" "CRONUS_SILU_FUSE_ROWS=16" "CRONUS_NORM_FUSE_ROWS=16 CRONUS_SILU_FUSE_ROWS=16"; do
    r=$(env $v python tools/timeline.py --n-dec $n --ctx 2142 --ppi-sms 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['pass_ms_reported'],4), d['kernels'])")
    echo "n=$n [$v] pass_ms kernels: $r"
  done
done 2>&1 | tee gpurun_out/fuse_ab.txt
