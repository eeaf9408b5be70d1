"""Multi-rank host logic of the compressed average on CPU (gloo, world size 2).

What a real run moves over NCCL is exercised here with torch.distributed on
CPU: every rank agrees on the fixed-capacity message layout computed by the
C library (no size exchange needed in count mode), a plain allgather of the
raw per-rank device messages delivers them in rank order, and decoding them
with the shard weights reproduces the reference's averaging step
(simulator.py:510-547) -- the oracle stands in for the GPU kernels, which the
-m gpu tests cover.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import message_layout, shard_weights

WORLD = 2
N = 3000
CHUNK = 1024


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rows():
    rng = np.random.default_rng(123)
    return rng.standard_normal((WORLD, N)) * 1e-2


def _worker(rank, port, theta, nm, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        rows = _rows()
        q = None if nm is None else F.tune_eps(-0.5, 0.5, *nm)
        lat = None if q is None else O.lattice(q.min, q.max, q.n_bits, q.mantissa_bits, q.eps)
        cfg = F.CodecConfig(F.SparsificationSpec(theta), q, chunk_size=CHUNK)
        n_chunks, nbytes, offs = message_layout(N, cfg)
        # 1. layout agreement across ranks
        lay = torch.tensor([n_chunks, nbytes, int(offs.sum())], dtype=torch.int64)
        allay = [torch.zeros_like(lay) for _ in range(WORLD)]
        dist.all_gather(allay, lay)
        assert all(torch.equal(allay[0], x) for x in allay)
        # 2. each rank's message in the device format, allgathered raw
        msg = O.compress(rows[rank], theta, "count", lat, False, CHUNK)
        dev = np.frombuffer(O.device_segments(msg, theta), dtype=np.uint8)
        assert dev.size == nbytes
        send = torch.from_numpy(dev.copy())
        recv = torch.empty(WORLD * nbytes, dtype=torch.uint8)
        dist.all_gather_into_tensor(recv, send)
        # 3. decode every rank's message, weighted sum in rank order
        w = shard_weights(7, WORLD)
        buf = recv.numpy().tobytes()
        got = sum(w[k] * O.decompress(O.from_device(buf[k * nbytes:(k + 1) * nbytes], N, CHUNK, theta, lat))
                  for k in range(WORLD))
        ref = O.average(rows, w, theta, "count", lat, False, CHUNK)
        out_q.put((rank, float(np.abs(got - ref).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("theta,nm", [(0.9, (8, 3)), (0.5, (6, 2)), (0.7, None)])
def test_two_rank_exchange_and_average(theta, nm):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, theta, nm, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    results = dict(q.get(timeout=10) for _ in range(WORLD))
    assert all(err <= 1e-12 for err in results.values()), results


def _agree_worker(rank, port, differ, out_q):
    from paper_1811_08596_b200.comm import check_config_agreement, config_fingerprint
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        # a quantizer calibrated per rank instead of once: rank 1's lattice differs
        q = F.tune_eps(-0.5, 0.5 if (rank == 0 or not differ) else 0.7, 8, 3)
        cfg = F.CodecConfig(F.SparsificationSpec(0.9), q, chunk_size=CHUNK)
        try:
            check_config_agreement(config_fingerprint(N, cfg, None, shard_weights(8, WORLD)))
            out_q.put((rank, "ok"))
        except ValueError as e:
            out_q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("differ", [False, True])
def test_config_agreement_across_ranks(differ):
    """GradientAverager refuses to average when the ranks' codec configs differ
    (every rank decodes the others' codes with its own lattice)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, port, differ, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = dict(q.get(timeout=10) for _ in range(WORLD))
    if differ:
        assert all("disagree" in v for v in res.values()), res
    else:
        assert all(v == "ok" for v in res.values()), res
