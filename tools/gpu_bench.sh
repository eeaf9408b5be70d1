#!/bin/bash
# usage: bash tools/gpu_bench.sh TAG [extra bench args]
TAG=${1:-r1}; shift
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
tail -3 gpurun_out/bench_$TAG.log; tail -3 gpurun_out/ncu_$TAG.log
