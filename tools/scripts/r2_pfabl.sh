for ab in 0 5 2 7; do echo "ablate=$ab"; CRONUS_PF_ABLATE=$ab python tools/prefill_probe.py --ctas -1 --shapes 448x1024,4096x0; done
CRONUS_PF_ABLATE=5 CRONUS_PF_PROBE=1 python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 1 2>&1 | tail -18 | head -10
