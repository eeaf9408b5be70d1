#!/bin/bash
# usage: bash tools/gpu_debug.sh "<pytest -k expr>"   (bounds-checked build, then pytest)
mkdir -p gpurun_out
export FGC_NVCC_FLAGS="-DFGC_BOUNDS"
python -m paper_1811_08596_b200.build > gpurun_out/dbg_build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$1" > gpurun_out/dbg.log 2>&1
echo "rc=$?" >> gpurun_out/dbg.log
grep -a "FGC_CHECK" gpurun_out/dbg.log | head; tail -5 gpurun_out/dbg.log
