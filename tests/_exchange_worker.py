"""Worker shared by the multi-process exchange tests (test_multigpu.py,
test_exchange_one_gpu.py): one rank of a compressed average over the peer
exchange or NCCL, checked against the oracle average of every rank's message
(simulator.py:520-547 with a real exchange).  Kept outside the test modules
so a module-level skip in one does not hide it from the other."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import torch


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, n, transport, mode, out_q, theta=0.9, nm=(8, 3), special=(), steps=4,
            same_gpu=False):
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
    # same_gpu: every rank on cuda:0 (the CUDA-IPC exchange works between
    # processes of one device; NCCL refuses duplicate GPUs, so no NCCL comm)
    torch.cuda.set_device(0 if same_gpu else rank)
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
        comm = (SimpleNamespace(rank=rank, world=world, group=None, handle=None, close=lambda: None)
                if same_gpu else NcclComm())
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
