# compute-sanitizer memcheck / racecheck / synccheck over the kernel tests (incl. the split
# prefill attention, the LPT decode plan and the CTA-pair GEMM) and a tiny serve.
# Summaries land in gpurun_out/san_*.log (condensed copies under profiles/r2_sanitizer/).
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 50 --error-exitcode 99"
K="attn_decode or attn_prefill or rmsnorm or qkv_rope or silu_mul or kv_copy or fused_rope"
G="test_gemm_store or test_gemm_splitk_red or silu_epilogue or silu_hybrid or fused_qkv"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool python -m pytest tests/test_kernels_gpu.py -q -k "$K" -p no:cacheprovider > gpurun_out/san_${tool}_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/san_${tool}_kernels.log
  timeout 1500 $CS --tool $tool python -m pytest tests/test_gemm_gpu.py -q -k "$G" -p no:cacheprovider > gpurun_out/san_${tool}_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/san_${tool}_gemm.log
  timeout 900 $CS --tool $tool python tools/sanitize_serve.py tiny > gpurun_out/san_${tool}_serve.log 2>&1; echo "rc=$?" >> gpurun_out/san_${tool}_serve.log
done
for f in gpurun_out/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
