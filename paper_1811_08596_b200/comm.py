"""Compressed gradient averaging across GPUs -- the exchange the reference
only simulates by value (simulator.py:510-547: per-worker
compress -> serialize -> deserialize -> decompress, then
``v_hat = shard_weights @ recon``).

One process per GPU.  Every rank compresses its own gradient into a
fixed-capacity device message (count mode: capacity is known a priori, so no
size exchange), one ``ncclAllGather`` moves all messages over NVLink /
NVSwitch, and every rank decodes all W messages, accumulates
``weight_w * X_w`` in the frequency domain in worker order and runs one
inverse FFT per chunk.  The result is identical on every rank.

Host-side logic (communicator bootstrap, layout agreement, weights) is
separate from the transport so it can be exercised with the gloo backend on
CPU (tests/test_comm_cpu.py).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .codec import CodecConfig, Plan, _desc

__all__ = ["message_layout", "shard_weights", "config_fingerprint", "check_config_agreement", "NcclComm",
           "PeerExchange", "GradientAverager", "allgather_average"]


def message_layout(n: int, config: CodecConfig) -> tuple[int, int, np.ndarray]:
    """(n_chunks, message_bytes, segment offsets) of the fixed-capacity
    device message for a gradient of length n -- host-only, no GPU."""
    spec = config.sparsification
    d = _desc(n, config.chunk_size, spec.theta, spec.mode, config.half_precision_pass, config.quantizer, False)
    nc = C.c_uint32()
    nb = C.c_uint64()
    _lib.check(_lib.lib.fgc_message_layout(C.byref(d), C.byref(nc), C.byref(nb), None))
    offs = np.zeros(nc.value + 1, dtype=np.uint64)
    _lib.check(_lib.lib.fgc_message_layout(C.byref(d), C.byref(nc), C.byref(nb), offs.ctypes.data))
    return int(nc.value), int(nb.value), offs


def shard_weights(batch_size: int, workers: int) -> np.ndarray:
    """simulator.py:481-485: worker w averages shard_sizes[w] examples of an
    np.array_split of the batch; weight = shard_size / batch_size."""
    sizes = np.array([len(p) for p in np.array_split(np.arange(batch_size), workers)])
    return sizes / batch_size


def config_fingerprint(n: int, config: CodecConfig, capacity_theta: float | None, weights) -> tuple:
    """What every rank of one averaging group must agree on: length, chunk,
    capacity theta (the message layout), mode, half pass, quantizer lattice,
    the shard weights and the peer-exchange transport (FGC_EXCHANGE_DIRECT:
    direct peer reads vs copy-engine pushes wait on different signals)."""
    q = config.quantizer
    spec = config.sparsification
    cap = spec.theta if capacity_theta is None else float(capacity_theta)
    return (int(n), int(config.chunk_size), cap, spec.mode, bool(config.half_precision_pass),
            None if q is None else (q.min, q.max, q.n_bits, q.mantissa_bits, q.eps),
            tuple(float(x) for x in np.asarray(weights, dtype=np.float64).reshape(-1)),
            os.environ.get("FGC_EXCHANGE_DIRECT", "0")[:1] or "0")


def check_config_agreement(fingerprint: tuple, group=None, world: int | None = None) -> None:
    """Every rank decodes every other rank's codes with its own plan and
    lattice: a rank with another quantizer, length or capacity would average
    garbage silently.  Compare fingerprints once, on all ranks (any
    torch.distributed backend); every rank raises the same ValueError."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if world is None else world
    allf = [None] * world
    dist.all_gather_object(allf, fingerprint, group=group)
    bad = [r for r, f in enumerate(allf) if f != allf[0]]
    if bad:
        raise ValueError(f"ranks {bad} disagree with rank 0 on the codec configuration (length, chunk, capacity "
                         f"theta, mode, quantizer, weights): every rank must average with the same config, e.g. a "
                         f"quantizer calibrated once and broadcast")


class NcclComm:
    """An NCCL communicator owned by libfgc_b200, bootstrapped through
    torch.distributed (any backend) by broadcasting the unique id."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            _lib.check(_lib.lib.fgc_nccl_unique_id(uid.ctypes.data))
        obj = [uid.tobytes()]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid = np.frombuffer(obj[0], dtype=np.uint8).copy()
        D.require_cuda()
        h = C.c_void_p()
        _lib.check(_lib.lib.fgc_nccl_comm_create(uid.ctypes.data, self.world, self.rank, C.byref(h)))
        self.handle = h

    def allgather(self, send: torch.Tensor, recv: torch.Tensor) -> None:
        _lib.check(_lib.lib.fgc_allgather(self.handle, send.data_ptr(), recv.data_ptr(), send.numel(), D.stream()))

    def allreduce_sum_(self, data: torch.Tensor) -> None:
        _lib.check(_lib.lib.fgc_allreduce_sum_f32(self.handle, data.data_ptr(), data.numel(), D.stream()))

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.lib.fgc_nccl_comm_destroy(self.handle)
            self.handle = None


class PeerExchange:
    """Double-buffered gather buffers shared with every peer through CUDA IPC:
    the copy engines move each rank's message pieces over NVLink while the
    codec kernels run (fgc_exchange_*; no collective kernels on the SMs).
    Handles are swapped through torch.distributed on ``group``."""

    def __init__(self, message_bytes: int, rank: int, world: int, group=None):
        import torch.distributed as dist
        D.require_cuda()
        self.rank, self.world = rank, world
        self._group = group
        self.handle = None
        # every step of the setup is agreed on by all ranks, so a failure on any
        # rank (no IPC, no stream memory operations) fails all of them alike
        h = C.c_void_p()
        mine, err = None, ""
        try:
            _lib.check(_lib.lib.fgc_exchange_create(world, rank, message_bytes, C.byref(h)))
            self.handle = h
            mine = np.zeros(128, dtype=np.uint8)
            _lib.check(_lib.lib.fgc_exchange_handles(h, mine.ctypes.data))
            mine = mine.tobytes()
        except Exception as e:                  # noqa: BLE001 -- reported below, on every rank
            err = f"rank {rank}: {e}"
        allh = [None] * world
        dist.all_gather_object(allh, (mine, err), group=group)
        errs = [e for _, e in allh if e]
        if not errs:
            try:
                buf = np.frombuffer(b"".join(m for m, _ in allh), dtype=np.uint8).copy()
                _lib.check(_lib.lib.fgc_exchange_open(h, buf.ctypes.data))
            except Exception as e:              # noqa: BLE001
                err = f"rank {rank}: {e}"
            oks = [None] * world
            dist.all_gather_object(oks, err, group=group)
            errs = [e for e in oks if e]
        if errs:
            if self.handle:
                _lib.lib.fgc_exchange_destroy(self.handle)
                self.handle = None
            raise RuntimeError("peer exchange unavailable: " + "; ".join(errs))
        dist.barrier(group)

    def close(self) -> None:
        if getattr(self, "handle", None):
            import torch.distributed as dist
            torch.cuda.synchronize()
            dist.barrier(self._group)          # no peer still reads our buffers
            _lib.lib.fgc_exchange_destroy(self.handle)
            self.handle = None


class GradientAverager:
    """Persistent buffers + plan for repeated compressed averaging of an
    n-element gradient: the per-step call allocates nothing and launches
    compress -> exchange -> decode-average on the current stream.

    transport "peer" (default; FGC_TRANSPORT overrides): pieces of the
    message move by peer-to-peer copies as soon as they are compressed and
    are decoded as they land (PeerExchange).  "nccl": one ncclAllGather.

    theta is a per-step argument (``step(grad, theta=...)``): the reference
    rebuilds its SparsificationSpec whenever the schedule moves theta
    (simulator.py:333-341, 522-528), here the plan, the message layout and
    the exchange stay.  Messages are sized for ``capacity_theta`` (default:
    the config's theta), the smallest drop ratio a step may ask for.

    Every averager owns its plan (device scratch, done tags, side stream): a
    plan is not safe on two streams at once (include/fgc_b200.h)."""

    def __init__(self, n: int, config: CodecConfig, weights, comm: NcclComm | None = None,
                 transport: str | None = None, capacity_theta: float | None = None):
        dev = D.require_cuda()
        spec = config.sparsification
        self.n = int(n)
        self.config = config
        self.comm = comm
        self.world = 1 if comm is None else comm.world
        w = np.asarray(weights, dtype=np.float64).reshape(-1)
        if w.size != self.world:
            raise ValueError(f"need one weight per rank ({self.world}), got {w.size}")
        self.weights = np.ascontiguousarray(w)
        cap = spec.theta if capacity_theta is None else float(capacity_theta)
        if not 0.0 <= cap <= spec.theta:
            raise ValueError(f"capacity_theta must be in [0, {spec.theta}], got {cap}")
        self.capacity_theta = cap
        self.plan = Plan(_desc(self.n, config.chunk_size, cap, spec.mode, config.half_precision_pass,
                               config.quantizer, False))
        self.theta = cap
        self.set_theta(spec.theta)
        self.message = self.plan.new_message()
        self.gathered = (torch.empty(self.world * self.plan.message_bytes, dtype=torch.uint8, device=dev)
                         if self.world > 1 else self.message)
        self.out = torch.empty(self.n, dtype=torch.float32, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)
        import os
        if self.world > 1:
            self._check_agreement(comm)
        self.transport = transport or os.environ.get("FGC_TRANSPORT", "peer")
        if self.transport not in ("peer", "nccl"):
            raise ValueError(f"unknown transport {self.transport!r}")
        self.exchange = None
        if self.world > 1 and self.transport == "peer":
            try:
                self.exchange = PeerExchange(self.plan.message_bytes, comm.rank, comm.world, comm.group)
            except RuntimeError as e:           # agreed on by every rank: all fall back together
                import warnings
                warnings.warn(f"{e}; using the NCCL allgather")
                self.transport = "nccl"

    def _check_agreement(self, comm) -> None:
        check_config_agreement(config_fingerprint(self.n, self.config, self.capacity_theta, self.weights),
                               comm.group, self.world)

    def close(self) -> None:
        if self.exchange is not None:
            self.exchange.close()
            self.exchange = None

    def set_theta(self, theta: float) -> None:
        """Drop ratio of the next steps (count mode: >= capacity_theta)."""
        theta = float(theta)
        if theta != self.theta:
            _lib.check(_lib.lib.fgc_plan_set_theta(self.plan.handle, theta, D.stream()))
            self.theta = theta

    def _check_out(self, out: torch.Tensor) -> torch.Tensor:
        if (not isinstance(out, torch.Tensor) or not out.is_cuda or out.device != self.out.device
                or out.dtype != torch.float32 or out.numel() != self.n or not out.is_contiguous()
                or out.data_ptr() % 8):
            raise ValueError("out must be a contiguous, 8-byte aligned float32 CUDA tensor of the planned "
                             "length on the averager's device")
        return out

    def step(self, grad: torch.Tensor, out: torch.Tensor | None = None, theta: float | None = None) -> torch.Tensor:
        """Average this rank's device gradient with every other rank's."""
        if grad.numel() != self.n or not grad.is_cuda:
            raise ValueError("gradient must be a CUDA tensor of the planned length")
        code = _lib.DTYPE_F64 if grad.dtype == torch.float64 else _lib.DTYPE_F32
        if grad.dtype not in (torch.float32, torch.float64):
            raise ValueError("gradient must be float32 or float64")
        if theta is not None:
            self.set_theta(theta)
        grad = D.aligned(grad.contiguous())
        dst = self.out if out is None else self._check_out(out)
        if self.exchange is not None:
            _lib.check(_lib.lib.fgc_exchange_average(self.plan.handle, self.exchange.handle, grad.data_ptr(), code,
                                                     self.weights.ctypes.data, dst.data_ptr(), self.flags.data_ptr(),
                                                     D.stream()))
            return dst
        comm = None if self.comm is None else self.comm.handle
        _lib.check(_lib.lib.fgc_allgather_average(self.plan.handle, comm, self.world, grad.data_ptr(), code,
                                                  self.weights.ctypes.data, self.message.data_ptr(),
                                                  self.gathered.data_ptr(), dst.data_ptr(), self.flags.data_ptr(),
                                                  D.stream()))
        return dst

    def step_host(self, grad: torch.Tensor, out: torch.Tensor | None = None, wait: bool = True,
                  theta: float | None = None) -> torch.Tensor:
        """The averaging step from and to host memory: the PCIe copies of the
        gradient and of the average overlap the codec kernels piece by piece
        (fgc_average_host).  Pass pinned CPU tensors for the overlap.  With
        wait=False the call returns once the work is queued on the current
        stream; synchronize it before reading `out`."""
        if grad.numel() != self.n or grad.is_cuda:
            raise ValueError("gradient must be a host tensor of the planned length")
        if grad.dtype not in (torch.float32, torch.float64):
            raise ValueError("gradient must be float32 or float64")
        code = _lib.DTYPE_F64 if grad.dtype == torch.float64 else _lib.DTYPE_F32
        grad = grad.contiguous()
        dst = out if out is not None else torch.empty(self.n, dtype=torch.float32, pin_memory=True)
        if dst.is_cuda or dst.numel() != self.n or dst.dtype != torch.float32 or not dst.is_contiguous():
            raise ValueError("out must be a contiguous float32 host tensor of the planned length")
        if theta is not None:
            self.set_theta(theta)
        dg = getattr(self, "_dgrad", None)
        if dg is None or dg.dtype != grad.dtype:
            dg = self._dgrad = torch.empty(self.n, dtype=grad.dtype, device=self.out.device)
        if self.world > 1 and self.exchange is None:
            # NCCL transport: plain copies around the device step
            dg.copy_(grad, non_blocking=True)
            dst.copy_(self.step(dg), non_blocking=True)
            if wait:
                torch.cuda.current_stream().synchronize()
            return dst
        x = self.exchange.handle if self.exchange is not None else None
        _lib.check(_lib.lib.fgc_average_host(self.plan.handle, x, grad.data_ptr(), code, self.weights.ctypes.data,
                                             dg.data_ptr(), self.message.data_ptr(), self.out.data_ptr(),
                                             dst.data_ptr(), self.flags.data_ptr(), D.stream()))
        if wait:
            torch.cuda.current_stream().synchronize()
        return dst

    def check(self) -> None:
        """Raise the reference's ValueError if any step saw a bad gradient."""
        f = D.read_flags(self.flags)
        if f:
            self.flags.zero_()
            D.raise_on_flags(f)


def allgather_average(local_grad, config: CodecConfig, weights, comm: NcclComm | None = None) -> np.ndarray:
    """One compressed averaging step (simulator.py:520-547 across real GPUs):
    returns ``sum_w weights[w] * decompress(compress(grad_w))`` as float64."""
    t, code = D.as_signal(local_grad)
    avg = GradientAverager(t.numel(), config, weights, comm)
    try:
        out = avg.step(t if t.dtype in (torch.float32, torch.float64) else t.float())
        avg.check()
        return out.double().cpu().numpy()
    finally:
        avg.close()
