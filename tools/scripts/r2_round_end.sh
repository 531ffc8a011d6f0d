# Round-end evidence: full GPU suite, smoke, the default bench line (CPU baseline included), the
# reference arm, and a clean ncu capture of the prefill attention at the mixed-pass shape
# (overlap off: the kernel with the partition's full CTA budget).
mkdir -p gpurun_out
T=${TAG:-r2z}
CRONUS_NO_PDL=1 CRONUS_ATTN_OVERLAP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_pp -s 40 -c 1 \
  -o gpurun_out/ncu2_prefill_pp_mixed -f python tools/one_pass.py --worker 1 --n-dec 80 --ctx 1440 --chunk 415 --pos0 1024 > gpurun_out/ncu2_a.log 2>&1
REF=1 TAG=$T bash tools/scripts/r2_full.sh
