"""The multi-process averaging step on ONE GPU: two ranks (two processes,
both on cuda:0) exchange their fused messages through the CUDA-IPC peer
exchange -- the same gather buffers, per-piece flags, copy-engine pushes and
in-kernel transports the multi-GPU runs use -- and each decodes both messages
in worker order (simulator.py:520-547).  Every rank's average must be within
1e-5 of the oracle average of both ranks' messages and bitwise equal across
ranks.  This is the exchange test a 1-GPU box can run; test_multigpu.py runs
the same worker across distinct GPUs (and over NCCL, which refuses two ranks
on one device)."""

import numpy as np
import pytest
import torch

from _exchange_worker import free_port, worker

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _run(n, transport, mode, theta=0.9, nm=(8, 3), special=(), steps=4, timeout=240):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, transport, mode, q, theta, nm, special, steps,
                                              True))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=timeout)
    hung = [p.pid for p in procs if p.is_alive()]
    for p in procs:                             # never leave a spinning rank behind
        if p.is_alive():
            p.kill()
            p.join(10)
    assert not hung, f"ranks {hung} did not finish in {timeout} s"
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(rel <= 1e-5 for _, rel, _ in res), res
    assert len({d for _, _, d in res}) == 1, "ranks disagree bitwise"


@pytest.mark.parametrize("transport,mode", [("peer", "count"), ("peer-direct", "count"), ("peer-kpush", "count"),
                                            ("peer", "energy")])
def test_two_ranks_one_gpu(transport, mode):
    """3 fused chunks + a 40960-sample generic tail, four steps with a
    different gradient and theta each, two of them through step_host."""
    _run(3 * 65536 + 40960, transport, mode)


def test_two_ranks_one_gpu_degenerate_chunks():
    """A zero chunk and a 1e-32-scaled chunk on rank 0, a (16, 9) lattice."""
    _run(5 * 65536 + 1234, "peer", "count", theta=0.97, nm=(16, 9), special=((0, 0.0), (3, 1e-32)))


def test_sixteen_chunks_two_ranks_one_gpu():
    """1M floats per rank (15 fused chunks + a generic tail), four steps."""
    _run(1_000_000, "peer", "count")
