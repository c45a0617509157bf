#!/bin/bash
# Round-1 profiling recipe (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dense_(kl|tv)" -s 4 -c 2 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
python scripts/micro_d2h.py > gpurun_out/micro.log 2>&1
tail -3 gpurun_out/ncu_full.log; cat gpurun_out/micro.log
