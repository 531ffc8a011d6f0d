# Prefill attention alone: CUDA-event timing at serve shapes, pipeline clock stamps of CTA 0,
# and one ncu --set full capture at the 448-token chunk / 1024 prefix shape.
mkdir -p gpurun_out
T=${TAG:-pf}
python tools/prefill_probe.py --shapes 448x1024,448x3072,2048x0,4096x0 > gpurun_out/${T}_probe.txt 2>&1
python tools/prefill_probe.py --ctas -1 --shapes 448x1024,448x3072,2048x0,4096x0 >> gpurun_out/${T}_probe.txt 2>&1
CRONUS_PF_PROBE=1 python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 1 > gpurun_out/${T}_stamps.txt 2>&1
CRONUS_PF_PROBE=1 python tools/prefill_probe.py --shapes 448x1024 --reps 1 >> gpurun_out/${T}_stamps.txt 2>&1
cat gpurun_out/${T}_probe.txt
if [ -z "$NONCU" ]; then
CRONUS_NO_PDL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_pp -s 5 -c 1 \
  -o gpurun_out/${T}_ncu -f python tools/prefill_probe.py --shapes 448x1024 --reps 1 > gpurun_out/${T}_ncu.log 2>&1
tail -3 gpurun_out/${T}_ncu.log
fi
