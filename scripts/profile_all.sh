#!/bin/bash
# ncu --set full captures of every product kernel family (run under gpurun).
#   bash scripts/profile_all.sh <tag>
TAG=${1:-r1}
mkdir -p gpurun_out
run() {  # name, kernel regex, skip, count, args...
  local name=$1 re=$2 skip=$3 cnt=$4; shift 4
  python scripts/prof_extras.py "$@" > gpurun_out/pa_${name}_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c $cnt \
      -o gpurun_out/prof_${name}_${TAG} python scripts/prof_extras.py "$@" \
      > gpurun_out/ncu_${name}_${TAG}.log 2>&1
  echo "$name rc=$?"
}
run csr "csr_(kl|tv)_kernel" 6 2 csr
run gemm "batched_kl_dmma2" 1 1 gemm
run tracer "trace_kernel" 1 1 tracer
run f32 "dense32_kernel" 6 2 f32
