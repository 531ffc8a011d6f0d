# Decode attention alone at the all-at-t=0 tail shapes (few sequences, 148 SMs): planner vs forced
# cluster sizes and ring depths; then the default bench line.
mkdir -p gpurun_out
S=3x2142,8x2142,16x2048
( for v in "X=1" "CRONUS_DEC_STAGES=2" "CRONUS_DEC_STAGES=4" "CRONUS_DEC_STAGES=6"; do
  echo "== $v"; env $v python tools/decode_bench.py --shapes $S 2>&1 | tail -3; done
  for c in 4 16; do echo "== cluster $c"; python tools/decode_bench.py --shapes $S --cluster $c 2>&1 | tail -3; done
  for s in 1 3 4; do echo "== slots/SM $s"; python tools/decode_bench.py --shapes $S --slots-per-sm $s 2>&1 | tail -3; done
) > gpurun_out/dec_small.txt 2>&1
cat gpurun_out/dec_small.txt
