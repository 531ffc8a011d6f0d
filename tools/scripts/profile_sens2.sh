for f in 1.0 0.75 0.5 0.35; do
  python - "$f" > gpurun_out/cfg_sens.cfg <<'PY'
import sys
a = float(sys.argv[1])
for ln in open("tests/golden/configs/b200_llama8b_coloc.cfg"):
    k = ln.split("=")[0].strip()
    if k == "low.prefill_k": ln = f"{k} = {float(ln.split('=')[1]) * a!r}\n"
    sys.stdout.write(ln)
PY
  timeout 900 python bench.py --config gpurun_out/cfg_sens.cfg --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'], d['cpi_busy_ms'], d['cpi_lent_iterations'])"
done
