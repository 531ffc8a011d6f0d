# Prefill attention key-split planner sweep (min sub-tiles per piece, max pieces per unit) at
# serve shapes on the full device and on the mixed-pass CTA budget (0.25 x 108 = 27).
S=448x1024,448x3072,415x1024,256x512,2048x0
for v in "X=1" "CRONUS_PF_MIN_PIECE=2" "CRONUS_PF_MIN_PIECE=8" "CRONUS_PF_MAX_PIECES=2" "CRONUS_PF_MAX_PIECES=8" "CRONUS_PF_MIN_PIECE=2 CRONUS_PF_MAX_PIECES=8"; do
  echo "== $v"; env $v python tools/prefill_probe.py --shapes $S 2>&1 | tail -5
  env $v python tools/prefill_probe.py --ctas 108 --shapes 448x1024,415x1024 2>&1 | tail -2
done
