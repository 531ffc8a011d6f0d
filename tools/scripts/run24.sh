# graph capture threshold sweep, then the whole GPU suite with graphs on (candidate default)
run() { env $1 CRONUS_GRAPH_STATS=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/b24.json 2> gpurun_out/b24.err
python -c "
import json; d=json.load(open('gpurun_out/b24.json')); print('$1', d['value'], d.get('ttft_p99_ms'), d.get('tbt_p99_ms'))"; grep "\[graphs\]" gpurun_out/b24.err | tail -1; }
for v in "CRONUS_GRAPHS=0" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=24" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=48" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=96" "CRONUS_GRAPHS=0" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=24" "CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=48"; do run "$v"; done
CRONUS_GRAPHS=1 CRONUS_GRAPH_MIN_SEEN=3 timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r24_pytest.log 2>&1; echo "pytest(graphs) rc=$?"; tail -2 gpurun_out/r24_pytest.log
