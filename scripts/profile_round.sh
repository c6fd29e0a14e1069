#!/bin/bash
# Profiling pass (run under gpurun on ONE GPU): launch list of the bench command + ncu --set full
# captures of the step kernel for the headline and the Adam workloads.  Outputs in gpurun_out/.
set -x
B="python bench.py --steps 30 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 3"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_resnet50_sgd.csv $B > gpurun_out/ncu_launches.log 2>&1
for w in resnet50_sgd gpt2_adamw vit_l16_adam_clip; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"step_tma|sumsq" -s 12 -c 3 \
      -o gpurun_out/prof_$w python bench.py --workload $w --steps 12 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 3 \
      > gpurun_out/ncu_full_$w.log 2>&1
done
