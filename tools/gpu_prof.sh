#!/bin/bash
# usage: bash tools/gpu_prof.sh TAG KERNEL_REGEX [prof_codec args]
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out
python tools/prof_codec.py "$@" > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 2 -o gpurun_out/prof_$TAG \
    python tools/prof_codec.py "$@" > gpurun_out/prof_ncu_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/prof_ncu_$TAG.log
tail -3 gpurun_out/prof_ncu_$TAG.log
