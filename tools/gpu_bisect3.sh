#!/bin/bash
# usage: bash tools/gpu_bisect3.sh N FLAGS...   (one build + dec_min per flag set)
mkdir -p gpurun_out
n=$1; shift
for F in "$@"; do
  export FGC_NVCC_FLAGS="$F"
  python -m paper_1811_08596_b200.build > /dev/null 2>&1
  echo "flags=[$F] $(CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/dec_min.py $n 2>&1 | tail -1)"
done
