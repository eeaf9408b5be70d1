#!/bin/bash
# usage: bash tools/gpu_multi.sh NGPUS TAG
NG=$1; TAG=$2
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$TAG.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider > gpurun_out/multi_$TAG.log 2>&1; echo "multi rc=$?" >> gpurun_out/multi_$TAG.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $NG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_n$NG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}_n$NG.log
tail -3 gpurun_out/multi_$TAG.log; tail -2 gpurun_out/bench_${TAG}_n$NG.log | cut -c1-1500
