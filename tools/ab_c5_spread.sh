#!/bin/bash
# config-5 run-to-run spread: the same bench line five times
source tools/gpu_ab.sh
export STEPS=5
for r in 1 2 3 4 5; do run c5_run$r 5 "" X=1; done
