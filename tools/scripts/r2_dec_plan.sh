# Decode planner check: small batches on 148 SMs and trace-length batches, engine planner only.
mkdir -p gpurun_out
( python tools/decode_bench.py --shapes 3x2142,8x2142,16x2048,24x2048,32x1400 2>&1 | tail -5
  python tools/decode_bench.py --trace-lens --shapes 16x0,32x0,64x0,97x0,128x0 2>&1 | tail -5 ) > gpurun_out/dec_plan.txt 2>&1
cat gpurun_out/dec_plan.txt
