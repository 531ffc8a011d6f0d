# Decode-pass timelines (CUPTI) at the all-at-t=0 tail shape (3 decoders, 148 SMs) and a
# 48-decoder pass on the 108-SM partition, with and without PDL, + kernel list JSON.
mkdir -p gpurun_out
python tools/timeline.py --n-dec 3 --ctx 2142 --ppi-sms 0 --json gpurun_out/tl_dec3.json > gpurun_out/tl_dec3.txt 2>&1
CRONUS_NO_PDL=1 python tools/timeline.py --n-dec 3 --ctx 2142 --ppi-sms 0 --json gpurun_out/tl_dec3_nopdl.json > gpurun_out/tl_dec3_nopdl.txt 2>&1
python tools/timeline.py --n-dec 48 --ctx 1400 --json gpurun_out/tl_dec48.json > gpurun_out/tl_dec48.txt 2>&1
CRONUS_GEMM_PROBE=1 python tools/one_pass.py --n-dec 3 --ctx 2142 > gpurun_out/gemm_probe_dec3.txt 2>&1
head -60 gpurun_out/tl_dec3.txt
