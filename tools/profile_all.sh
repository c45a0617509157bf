#!/bin/bash
# ncu --set full captures of every product kernel family (run under gpurun).
#   bash tools/profile_all.sh <tag> [comma list: csr,gemm,gemm_i8,tracer,f32,hausdorff]
TAG=${1:-r1}
mkdir -p gpurun_out
run() {  # name, kernel regex, skip, count, args...
  local name=$1 re=$2 skip=$3 cnt=$4; shift 4
  python tools/prof_extras.py "$@" > gpurun_out/pa_${name}_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c $cnt \
      -o gpurun_out/prof_${name}_${TAG} python tools/prof_extras.py "$@" \
      > gpurun_out/ncu_${name}_${TAG}.log 2>&1
  echo "$name rc=$?"
}
ONLY=${2:-csr,gemm,gemm_i8,tracer,f32,hausdorff}
want() { [[ ",$ONLY," == *",$1,"* ]]; }
want csr && run csr "csr_(kl|tv)_kernel|csr_kl_fixup_queue" 9 3 csr
want gemm && run gemm "batched_kl_dmma2" 1 1 gemm
want gemm_i8 && run gemm_i8 "batched_kl_i8|slice_(rows|targets)" 0 3 gemm_i8
want tracer && run tracer "trace_kernel" 1 1 tracer
want f32 && run f32 "dense32_kernel" 6 2 f32
want hausdorff && run hausdorff "hausdorff_kernel|polyline" 0 3 hausdorff
