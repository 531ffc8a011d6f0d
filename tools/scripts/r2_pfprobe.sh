export CRONUS_PF_PROBE=1
python tools/prefill_probe.py --ctas -1 --shapes 64x1024 --reps 1 2>&1 | tail -22
python tools/prefill_probe.py --ctas -1 --shapes 448x1024 --reps 1 2>&1 | tail -20
