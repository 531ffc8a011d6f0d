# Session-5 final: GPU suite + smoke + default bench (+ reference arm), ncu --set full of the
# production prefill kernel at 448 @ 1024 after the batched-issue change.
mkdir -p gpurun_out
REF=1 TAG=r2s10 bash tools/scripts/r2_full.sh
CRONUS_NO_PDL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_pp -s 5 -c 1 \
  -o gpurun_out/s5_ncu_prefill_448x1024_batched -f python tools/prefill_probe.py --shapes 448x1024 --reps 1 > gpurun_out/s5_ncu_d.log 2>&1
ls -la gpurun_out/*.ncu-rep
