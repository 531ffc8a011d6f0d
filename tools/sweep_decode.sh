#!/bin/bash
# Dev: decode-attention split-size sweep via CRONUS_DECODE_WAVES (kernel_probe decode cases)
for w in 1 2 4 8; do echo "waves=$w"; CRONUS_DECODE_WAVES=$w timeout 120 python tools/kernel_probe.py --only decode 2>&1 | tail -8; done
