#!/bin/bash
# Profiling recipe (run under gpurun from the repo root):
#   bash tools/profile_round.sh <tag> [bench args...]
# 1) plain bench run, 2) ncu launch list of the same command,
# 3) ncu --set full of the dense KL/TV kernels (same command again).
TAG=${1:-r1}; shift
ARGS=${@:-"--steps 3 --warmup 3 --no-cpu"}
mkdir -p gpurun_out
CMD="python bench.py $ARGS"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dense_(kl|tv)_kernel" -s 4 -c 2 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile $TAG done"; tail -2 gpurun_out/ncu_full_$TAG.log
