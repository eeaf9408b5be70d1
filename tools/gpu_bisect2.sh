#!/bin/bash
# usage: bash tools/gpu_bisect2.sh "<pytest -k expr>" FLAGS...   (one build + test per flag set)
mkdir -p gpurun_out
K=$1; shift
for F in "$@"; do
  export FGC_NVCC_FLAGS="$F"
  python -m paper_1811_08596_b200.build > /dev/null 2>&1
  CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/bis_log.txt 2>&1
  echo "flags=[$F] rc=$? $(grep -a -o 'NativeError.*' gpurun_out/bis_log.txt | head -1 | cut -c1-150) $(tail -1 gpurun_out/bis_log.txt)"
done
