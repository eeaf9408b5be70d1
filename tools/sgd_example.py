"""Data-parallel SGD with compressed gradient averaging on GPUs (BASELINE.json
config 5 shape: a ResNet-32-sized parameter vector, ~464K floats), using the
reference simulator's coupled diminishing theta schedule
(simulator.py:333-341: theta_t = min(cap, sqrt(L * eta_t))) and its
diminishing learning rate (eta_t = eta0 / (1 + t/tau)**power).

Each rank owns a shard of a synthetic least-squares problem
f(x) = 1/(2m) ||A x - b||^2 over its rows; per step it computes its shard
gradient on the GPU, the GradientAverager averages the W compressed
gradients (compress -> peer exchange -> frequency-domain weighted decode),
and every rank applies the identical update.  One averager (one plan, one
peer exchange) serves the whole schedule: its messages are sized for
capacity_theta = 0 and every step passes its theta at run time.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/sgd_example.py --iters 200
    python tools/sgd_example.py --iters 200            # single GPU
"""
import argparse
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager, NcclComm, shard_weights


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=464_154)
    ap.add_argument("--rows", type=int, default=256, help="rows of A per rank")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--eta0", type=float, default=None, help="default 1/(2L)")
    ap.add_argument("--tau", type=float, default=100.0)
    ap.add_argument("--power", type=float, default=1.0)
    ap.add_argument("--cap", type=float, default=0.99)
    ap.add_argument("--nbits", type=int, default=8)
    ap.add_argument("--mantissa", type=int, default=3)
    ap.add_argument("--passthrough", action="store_true", help="no quantizer (raw float32 codes)")
    a = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
        comm = NcclComm()
    dev = torch.device("cuda")
    gen = torch.Generator(dev).manual_seed(1234 + rank)
    A = torch.randn(a.rows, a.dim, device=dev, generator=gen) / math.sqrt(a.dim)
    x_star = torch.randn(a.dim, device=dev, generator=torch.Generator(dev).manual_seed(7))
    b = A @ x_star
    # L = largest eigenvalue of A^T A / rows (power iteration; identical on every rank after averaging)
    v = torch.randn(a.dim, device=dev, generator=torch.Generator(dev).manual_seed(9))
    for _ in range(30):
        v = A.T @ (A @ v) / a.rows
        v = v / v.norm()
    L = float(v @ (A.T @ (A @ v)) / a.rows)
    if world > 1:
        t = torch.tensor([L], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        L = float(t)
    eta0 = a.eta0 or 1.0 / (2.0 * L)
    w = shard_weights(world * a.rows, world)
    x = torch.zeros(a.dim, device=dev)
    q = None
    avg = None
    trace = []
    for t in range(a.iters):
        eta = eta0 / (1.0 + t / a.tau) ** a.power
        theta = min(a.cap, math.sqrt(L * eta))
        g = A.T @ (A @ x - b) / a.rows
        if q is None and not a.passthrough:
            # one range for every rank, fixed from rank 0's first gradient
            # (TrainConfig.quantizer, simulator.py:354): ranks decode each
            # other's codes with it
            g0 = g.clone()
            if world > 1:
                torch.distributed.broadcast(g0, src=0)
            q = F.calibrate([g0], a.nbits, a.mantissa)
        if avg is None:
            avg = GradientAverager(a.dim, F.CodecConfig(F.SparsificationSpec(theta), q), w, comm,
                                   capacity_theta=0.0)
        v_hat = avg.step(g, theta=theta)
        x = x - eta * v_hat
        if t % 20 == 0 or t == a.iters - 1:
            loss = float(((A @ x - b) ** 2).mean() / 2)
            trace.append({"t": t, "theta": theta, "eta": eta, "shard_loss": loss})
    avg.check()
    avg.close()
    if rank == 0:
        print(json.dumps({"world": world, "dim": a.dim, "L": L, "trace": trace}), flush=True)
    if comm is not None:
        comm.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
