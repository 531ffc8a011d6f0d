# Mixed pass (435-token chunk at 1024 + 77 decoders, 108 SMs): GEMM variants, per-kernel times.
for v in "X=1" "CRONUS_SILU_HYBRID=0" "CRONUS_GEMM_PAIR=0" "CRONUS_QKV_STREAMK=0"; do
  env $v python tools/timeline.py --n-dec 77 --ctx 1447 --chunk 435 --pos0 1024 --json gpurun_out/tl_mix_ab.json > /dev/null 2>&1
  python - "$v" <<'PY'
import json, sys
d = json.load(open('gpurun_out/tl_mix_ab.json')); ks = d['kernels']
i0 = [i for i, k in enumerate(ks) if 'embed' in k[2]][-1]
g = [round(e - s, 1) for s, e, c in ks[i0 + 1:i0 + 60] if 'gemm' in c][:8]
print(sys.argv[1], 'pass_ms', round(d['summary']['pass_ms_reported'], 3), 'gemm durations layer 1-2', g)
PY
done
