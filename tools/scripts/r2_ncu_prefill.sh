# ncu --set full (with source) of the prefill attention kernel alone at the C2 chunk shape.
mkdir -p gpurun_out
export CRONUS_NO_PDL=1
N="timeout 600 ncu --set full --clock-control none --import-source on"
$N -k regex:attn_prefill_pp -s 5 -c 1 -o gpurun_out/ncu_pf_448x1024_split -f python tools/prefill_probe.py --ctas 108 --shapes 448x1024 --reps 2 > gpurun_out/ncu_pf1.log 2>&1
$N -k regex:attn_prefill_pp -s 5 -c 1 -o gpurun_out/ncu_pf_448x1024_nosplit -f python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 2 > gpurun_out/ncu_pf2.log 2>&1
$N -k regex:attn_prefill_pp -s 5 -c 1 -o gpurun_out/ncu_pf_4096x0 -f python tools/prefill_probe.py --ctas -1 --shapes 4096x0 --reps 2 > gpurun_out/ncu_pf3.log 2>&1
ls -la gpurun_out/ncu_pf_*
