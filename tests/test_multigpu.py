"""Compressed average across real GPUs: the fixed-capacity device messages
move over NVLink (peer-to-peer copies through CUDA IPC, or one NCCL
allgather), then every rank decodes the W messages in worker order
(simulator.py:520-547 with a real exchange).  Needs >= 2 GPUs; the 2-rank
host logic is covered on CPU by test_comm_cpu.py."""

import numpy as np
import pytest
import torch

from _exchange_worker import free_port, worker

pytestmark = pytest.mark.gpu

if torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)


@pytest.mark.parametrize("transport,mode", [("peer", "count"), ("peer-direct", "count"), ("peer-kpush", "count"),
                                            ("nccl", "count"),
                                            ("peer", "energy"), ("nccl", "energy")])
@pytest.mark.parametrize("n", [3 * 65536 + 40960, 1_000_000])
def test_compressed_average_two_ranks(n, transport, mode):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, transport, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(rel <= 1e-5 for _, rel, _ in res), res
    assert len({d for _, _, d in res}) == 1, "ranks disagree bitwise"


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_c2_full_size_two_ranks(transport):
    """BASELINE config 2 at its full size (25.6M floats per rank, 391 fused
    chunks + the 40960-sample tail) over the exchange: 2 steps with different
    gradients and theta; every rank's average within 1e-5 of the oracle
    average of both ranks' messages, and bitwise equal across ranks."""
    import torch.multiprocessing as mp
    world, n = 2, 25_600_000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, transport, "count", q, 0.9, (8, 3), (), 2))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(rel <= 1e-5 for _, rel, _ in res), res
    assert len({d for _, _, d in res}) == 1, "ranks disagree bitwise"


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("transport,mode", [("peer", "count"), ("peer-direct", "count"), ("peer-kpush", "count"),
                                            ("nccl", "count"), ("peer", "energy")])
def test_compressed_average_four_ranks(transport, mode):
    """The same steps on 4 ranks: every rank decodes 4 messages in worker
    order; results within 1e-5 of the oracle average and bitwise equal."""
    import torch.multiprocessing as mp
    world, n = 4, 5 * 65536 + 40960
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, transport, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=400)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(rel <= 1e-5 for _, rel, _ in res), res
    assert len({d for _, _, d in res}) == 1, "ranks disagree bitwise"


@pytest.mark.parametrize("transport", ["peer", "peer-direct", "peer-kpush"])
@pytest.mark.parametrize("seed", range(4))
def test_random_configs_two_ranks(seed, transport):
    """Random sizes, keep ratios and lattices over the peer exchange, with
    degenerate chunks on one rank."""
    import torch.multiprocessing as mp
    rng = np.random.default_rng(70 + seed)
    n = int(rng.integers(1, 120)) * 65536 + int(rng.integers(0, 65536))
    theta = float(rng.choice([0.5, 0.9, 0.97]))
    nm = [(8, 3), (4, 2), (16, 9)][int(rng.integers(0, 3))]
    special = ((0, 0.0), (int(rng.integers(0, n // 65536)), 1e-32))
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, transport, "count", q, theta, nm, special))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(rel <= 1e-5 for _, rel, _ in res), (res, n, theta, nm)
    assert len({d for _, _, d in res}) == 1, "ranks disagree bitwise"
