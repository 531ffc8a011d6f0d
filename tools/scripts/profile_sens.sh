# Sensitivity of req/s to the CPI cost profile the balancer plans with.
C=tests/golden/configs/b200_llama8b_coloc.cfg
for v in "1 1 1" "0.5 1 1" "2 1 1" "1 1 0.5" "1 1 2"; do
  set -- $v
  python - "$1" "$2" "$3" > gpurun_out/cfg_sens.cfg <<'PY'
import sys
a, b, c = map(float, sys.argv[1:4])
for ln in open("tests/golden/configs/b200_llama8b_coloc.cfg"):
    k = ln.split("=")[0].strip()
    if k == "high.chunked_k_ctxp": ln = f"{k} = {float(ln.split('=')[1]) * a!r}\n"
    if k == "high.chunked_k_ctxd": ln = f"{k} = {float(ln.split('=')[1]) * b!r}\n"
    if k == "high.chunked_b": ln = f"{k} = {float(ln.split('=')[1]) * c!r}\n"
    sys.stdout.write(ln)
PY
  timeout 900 python bench.py --config gpurun_out/cfg_sens.cfg --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'])"
done
