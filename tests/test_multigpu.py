"""Compressed average across real GPUs: the fixed-capacity device messages
move over NVLink (peer-to-peer copies through CUDA IPC, or one NCCL
allgather), then every rank decodes the W messages in worker order
(simulator.py:520-547 with a real exchange).  Needs >= 2 GPUs; the 2-rank
host logic is covered on CPU by test_comm_cpu.py."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, transport, mode, out_q, theta=0.9, nm=(8, 3), special=(), steps=4):
    import torch.distributed as dist

    import oracle as O
    import paper_1811_08596_b200 as F
    from paper_1811_08596_b200.comm import GradientAverager, NcclComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # "peer": copy-engine pushes into a local gather buffer; "peer-direct":
    # the decode reads the peers' fused segments in place over NVLink;
    # "peer-kpush": the compress kernel stores its segments into the peers'
    os.environ["FGC_EXCHANGE_DIRECT"] = {"peer-direct": "1", "peer-kpush": "2"}.get(transport, "0")
    transport = "peer" if transport.startswith("peer") else transport
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        thetas = [theta, min(1.0, theta + 0.02), theta, min(1.0, theta + 0.05)][:steps]
        rows = []                                # a different gradient on every step and rank
        for s in range(steps):
            rng = np.random.default_rng(77 + s)
            r = (rng.standard_normal((world, n)) * 1e-2).astype(np.float32)
            for c, scale in special:            # zero / tiny chunks on rank 0
                r[0, c * 65536:(c + 1) * 65536] *= scale
            rows.append(r)
        q = F.calibrate([rows[0][0]], *nm)
        cfg = F.CodecConfig(F.SparsificationSpec(theta, mode), q)
        comm = NcclComm()
        w = F.shard_weights(5 * world + 1, world)
        avg = GradientAverager(n, cfg, w, comm, transport=transport)
        outs = []
        for s in range(steps):                  # the peer exchange alternates two gather buffers
            g = torch.from_numpy(rows[s][rank]).cuda()
            outs.append(avg.step(g, theta=thetas[s]).clone())
        for s in [s for s in (1, 2) if s < steps]:   # host-buffer step: same bits as the device step
            hout = avg.step_host(torch.from_numpy(rows[s][rank]).pin_memory(), theta=thetas[s])
            assert torch.equal(hout, outs[s].cpu()), "host step disagrees"
        avg.check()
        if transport == "peer" and mode == "energy" and avg.exchange is not None:
            # energy messages are sized for every slot; only the used bytes travel
            import ctypes
            from paper_1811_08596_b200 import _lib
            f = _lib.lib.fgc_debug_exchange_pushed
            f.restype, f.argtypes = ctypes.c_ulonglong, [ctypes.c_void_p]
            pushed = f(avg.exchange.handle)
            full = (steps + 2) * avg.plan.message_bytes * (world - 1)
            assert 0 < pushed < full, (pushed, full)
        avg.close()
        # oracle: decode every rank's message of every step (the wire bytes of a
        # rank's compress are bit-identical on all ranks, so serialize locally)
        rels = []
        for s in range(steps):
            scfg = F.CodecConfig(F.SparsificationSpec(thetas[s], mode), q)
            msgs = [F.compress(rows[s][k], scfg) for k in range(world)]
            ref = sum(w[k] * O.decompress(O.from_wire(F.serialize(msgs[k]))) for k in range(world))
            got = outs[s].double().cpu().numpy()
            # a coarse lattice can zero every code (eps above every coefficient): then got must be 0 too
            rels.append(float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)))
        # every rank must hold bit-identical results
        digest = float(sum(np.frombuffer(o.cpu().numpy().tobytes(), dtype=np.uint32).astype(np.float64).sum()
                           for o in outs))
        out_q.put((rank, max(rels), digest))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport,mode", [("peer", "count"), ("peer-direct", "count"), ("peer-kpush", "count"),
                                            ("nccl", "count"),
                                            ("peer", "energy"), ("nccl", "energy")])
@pytest.mark.parametrize("n", [3 * 65536 + 40960, 1_000_000])
def test_compressed_average_two_ranks(n, transport, mode):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, transport, mode, q)) for r in range(world)]
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
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, transport, "count", q, 0.9, (8, 3), (), 2))
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
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, transport, mode, q)) for r in range(world)]
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
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, transport, "count", q, theta, nm, special))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(rel <= 1e-5 for _, rel, _ in res), (res, n, theta, nm)
    assert len({d for _, _, d in res}) == 1, "ranks disagree bitwise"
