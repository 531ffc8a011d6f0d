# cluster planner residency assumption (CRONUS_DEC_SLOTS_PER_SM) with the per-launch ring depth
for r in 2 3 2 3; do CRONUS_DEC_SLOTS_PER_SM=$r timeout 300 python tools/pass_sweep.py llama3-8b 4x2048 8x2048 12x2048 16x2048 24x2048 32x2048 48x1024 76x1024 2>&1 | tail -1 | sed "s/^/slots=$r /"; done
