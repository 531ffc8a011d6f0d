# Mixed passes: prefill-attention CTA share while the decode attention runs on the side stream.
for n in "77 1447 435 1024" "55 1260 457 2048" "30 1250 482 512"; do
  set -- $n
  for v in 0.15 0.25 0.35 0.5; do
    r=$(CRONUS_ATTN_OVERLAP=$v python tools/timeline.py --n-dec $1 --ctx $2 --chunk $3 --pos0 $4 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['pass_ms_reported'],4))")
    echo "dec=$1 chunk=$3@$4 overlap=$v pass_ms=$r"
  done
done
