# CUDA-graph replay of decode passes with capture on the N-th sighting (CRONUS_GRAPH_MIN_SEEN)
CRONUS_GRAPH_MIN_SEEN=3 timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -x -q -k graph 2>&1 | tail -2
run() { env $1 CRONUS_GRAPH_STATS=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b23.json 2> gpurun_out/b23.err
python -c "
import json; d=json.load(open('gpurun_out/b23.json')); print('$1', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'))"; grep "\[graphs\]" gpurun_out/b23.err | tail -1; }
for v in "CRONUS_GRAPHS=0" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=2" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=8" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=24" "CRONUS_GRAPHS=0" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=8"; do run "$v"; done
