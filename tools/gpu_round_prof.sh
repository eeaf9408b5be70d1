#!/bin/bash
# usage: bash tools/gpu_round_prof.sh TAG -- full bench line, launch list, ncu --set full of the fused kernels
TAG=${1:-r1}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full_$TAG.log
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/prof_codec.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o gpurun_out/prof_$TAG \
    python tools/prof_codec.py > gpurun_out/prof_ncu_$TAG.log 2>&1
echo "prof rc=$?" >> gpurun_out/prof_ncu_$TAG.log
tail -2 gpurun_out/bench_full_$TAG.log | cut -c1-600; tail -2 gpurun_out/prof_ncu_$TAG.log
