# Decode planner check: small batches on 148 SMs and trace-length batches, engine planner only.
mkdir -p gpurun_out
( python tools/decode_bench.py --shapes 1x2142,2x2142,3x2142,4x2142,1x8192,8x2142,16x2048,24x2048,32x1400 2>&1 | tail -9
  python tools/decode_bench.py --trace-lens --shapes 4x0,16x0,32x0,64x0,97x0,128x0 2>&1 | tail -6 ) > gpurun_out/dec_plan.txt 2>&1
cat gpurun_out/dec_plan.txt
