for B in 512 1024 2048; do
  sed "s/^max_batched_tokens_high = .*/max_batched_tokens_high = $B/" tests/golden/configs/b200_llama8b_coloc.cfg > gpurun_out/cfg_B.cfg
  timeout 900 python bench.py --config gpurun_out/cfg_B.cfg --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$B', d['value'], d['ttft_p99_ms'], d['tbt_p99_ms'], d['cpi_iterations'])"
done
