#!/bin/bash
# config-5 run-to-run spread: clock sampling interval (nvidia-smi NVML queries during the
# host-bound timed region) and worker count
source tools/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export STEPS=5
for r in 1 2 3; do
  run c5_clk100_$r 5 "" X=1
  run c5_clk0_$r 5 "--clock-ms 0" X=1
  run c5_clk1000_$r 5 "--clock-ms 1000" X=1
done
for r in 1 2; do run c5_w1_clk0_$r 5 "--clock-ms 0 --workers 1" X=1; run c5_w8_clk0_$r 5 "--clock-ms 0 --workers 8" X=1; done
