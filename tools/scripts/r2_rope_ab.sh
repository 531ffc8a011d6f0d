# RoPE/append metadata hoisted before the dependency wait: kernel + engine parity, mixed-pass time.
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "rope or prefill" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do
python tools/timeline.py --n-dec 77 --ctx 1447 --chunk 435 --pos0 1024 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); c=d['classes'].get('qkv_rope_append_kernel',{})
print('mixed pass_ms', round(d['pass_ms_reported'],4), 'rope', c)"
done
