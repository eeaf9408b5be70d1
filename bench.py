"""Benchmark: gradient GB/s through compress + allgather + decompress/average
(BASELINE.json `metric`) on synthetic ResNet-50-sized gradients.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = every rank compresses its own n-float gradient (weak scaling),
allgathers the fixed-capacity messages over NCCL, and decodes the weighted
average of all W messages (frequency-domain accumulate + one iFFT per chunk).

value : whole-job GB/s = W * 4n bytes / (max-over-ranks device time of one
        step), inputs resident in HBM, L2 flushed (256 MB write) between
        timed steps, CUDA events on the launching stream.
e2e   : same metric through the public API with pinned host buffers: H2D of
        the gradient, the step, D2H of the averaged gradient, all timed.
--impl reference: the reference's CPU implementation of the path (the oracle
        port, chunk-parallel over all host cores), rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # BASELINE.json configs[1]: ResNet-50-sized gradient, keep 0.1 (reference theta=0.9 drop), 8-bit range float
    "resnet50": dict(n=25_600_000, theta=0.9, n_bits=8, mbits=3, chunk=65536),
    "cpu1m": dict(n=1_000_000, theta=0.9, n_bits=8, mbits=3, chunk=65536),
    "alexnet": dict(n=61_000_000, theta=0.9, n_bits=8, mbits=3, chunk=65536),
    "vgg16": dict(n=138_000_000, theta=0.9, n_bits=8, mbits=3, chunk=65536),
}
METRIC = "gradient GB/s through compress+sync+decompress; sync ms/step at 1/2/4/8 B200"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML every
    2 ms while the timed region runs (the same fields as the nvidia-smi
    clocks line of the profiling recipe)."""

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.rows = []
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=1)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        nv = self.nv
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
        reasons = sorted({n for _, rs in self.rows for bit, n in names.items() if rs & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


# ---------------------------------------------------------------- reference arm

def _ref_chunk_job(args):
    g_bytes, theta, lat, chunk, mode = args
    import oracle as O
    g = np.frombuffer(g_bytes, dtype=np.float32).astype(np.float64)
    msg = O.compress(g, theta, mode, lat, False, chunk)
    wire = O.to_wire(msg)
    return O.decompress(O.from_wire(wire))


def cpu_reference(wl: dict, seconds_budget: float, cores: int | None = None, sample_chunks: int | None = None):
    """The reference CPU path (oracle port of compress -> serialize ->
    deserialize -> decompress), chunk-parallel over `cores` processes on a
    bounded sample of the workload.  Returns (GB/s, cores, sample desc)."""
    import multiprocessing as mp

    import oracle as O
    cores = cores or len(os.sched_getaffinity(0))
    chunk = wl["chunk"]
    rng = np.random.default_rng(0)
    probe = (rng.standard_normal(chunk) * 1e-2).astype(np.float32)
    lat = O.calibrate([probe], wl["n_bits"], wl["mbits"])
    t0 = time.perf_counter()
    mode = wl.get("mode", "count")
    _ref_chunk_job((probe.tobytes(), wl["theta"], lat, chunk, mode))
    per_chunk = time.perf_counter() - t0
    if sample_chunks is None:
        sample_chunks = int(max(cores, min(wl["n"] // chunk, seconds_budget * cores / max(per_chunk, 1e-3))))
    g = (rng.standard_normal(sample_chunks * chunk) * 1e-2).astype(np.float32)
    jobs = [(g[i * chunk:(i + 1) * chunk].tobytes(), wl["theta"], lat, chunk, mode) for i in range(sample_chunks)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        t0 = time.perf_counter()
        pool.map(_ref_chunk_job, jobs, chunksize=max(1, sample_chunks // (4 * cores)))
        dt = time.perf_counter() - t0
    gbs = 4.0 * sample_chunks * chunk / dt / 1e9
    return gbs, cores, f"{sample_chunks} chunks x {chunk} floats ({sample_chunks * chunk} floats), {dt:.2f}s"


def host_info() -> dict:
    """CPU model, numpy version and SIMD dispatch line (BASELINE.md section 4
    step 2), plus the H1 self-check: numpy's complex128 abs on THIS host
    equals the cabs formula the selection key follows."""
    import platform
    info = {"numpy": np.__version__, "python": platform.python_version()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        from numpy._core import _multiarray_umath as mu
        feats = mu.__cpu_features__
        info["simd"] = {"baseline": list(mu.__cpu_baseline__),
                        "found": [k for k in mu.__cpu_dispatch__ if feats.get(k)],
                        "not_found": [k for k in mu.__cpu_dispatch__ if not feats.get(k)]}
    except Exception as e:                          # noqa: BLE001
        info["simd"] = f"unavailable: {e}"
    try:
        import oracle as O
        rng = np.random.default_rng(11)
        re = rng.standard_normal(20000) * np.exp2(rng.integers(-40, 40, 20000))
        im = re * np.exp2(rng.integers(-30, 30, 20000)) * rng.choice([-1, 1], 20000)
        im[:100] = 0.0
        got = np.abs(re + 1j * im)
        want = np.array([O.magnitude_exact(a, b) for a, b in zip(re, im)])
        info["h1_cabs_selfcheck"] = {"values": int(re.size), "mismatches": int(np.count_nonzero(got != want))}
    except Exception as e:                          # noqa: BLE001
        info["h1_cabs_selfcheck"] = f"error: {e}"
    return info


def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    steps = []
    cores = len(os.sched_getaffinity(0))
    for i in range(args.warmup + args.steps):
        gbs, cores, sample = cpu_reference(wl, seconds_budget=max(2.0, 20.0 / max(1, args.steps)), cores=cores)
        if i >= args.warmup:
            steps.append(gbs)
    v = statistics.median(steps)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 4.0 * wl["n"] / (v * 1e9) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic gaussian sigma=1e-2",
            "config": workload_config(args, wl, world),
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample,
                             "host": host_info()},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, wl, world):
    mode = wl.get("mode", "count")
    keep = (f"keep={1 - wl['theta']:.2f} (reference theta_drop={wl['theta']})" if mode == "count" else
            f"energy mode, theta={wl['theta']} (drop while cumulative energy <= theta^2 of the total)")
    return {"workload": f"{args.workload}: n={wl['n']} floats, {keep}, {wl['n_bits']}-bit range float "
                        f"m={wl['mbits']}, chunk={wl['chunk']}, W={world} ranks",
            "mode": mode,
            "n": wl["n"], "theta_drop": wl["theta"], "n_bits": wl["n_bits"], "mantissa_bits": wl["mbits"],
            "chunk_size": wl["chunk"], "world": world, "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MB write)"}


# ---------------------------------------------------------------- our arm

def run_ours(args, wl, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1811_08596_b200 as F
    from paper_1811_08596_b200.comm import GradientAverager, NcclComm

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = wl["n"]
    # quantizer calibrated once on rank 0's gradient (every rank regenerates it)
    g0 = torch.randn(n, device=dev, generator=torch.Generator(dev).manual_seed(1000)) * 1e-2
    q = F.calibrate([g0], wl["n_bits"], wl["mbits"])
    del g0
    cfg = F.CodecConfig(F.SparsificationSpec(wl["theta"], wl.get("mode", "count")), q, chunk_size=wl["chunk"])
    grad = torch.randn(n, device=dev, generator=torch.Generator(dev).manual_seed(1000 + rank)) * 1e-2
    comm = NcclComm() if world > 1 else None
    weights = np.full(world, 1.0 / world)
    avg = GradientAverager(n, cfg, weights, comm, transport=args.transport)
    M = avg.plan.message_bytes
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timing, per-stage events
    from paper_1811_08596_b200 import _lib, _device as D
    import ctypes as C

    def one_step(ev=None):
        if ev is None:
            avg.step(grad)
            return
        ev[0].record()
        _lib.check(_lib.lib.fgc_compress(avg.plan.handle, grad.data_ptr(), _lib.DTYPE_F32, avg.message.data_ptr(),
                                         avg.flags.data_ptr(), D.stream()))
        ev[1].record()
        if world > 1:
            comm.allgather(avg.message, avg.gathered)
        ev[2].record()
        _lib.check(_lib.lib.fgc_decode_average(avg.plan.handle, avg.gathered.data_ptr(), world, M,
                                               avg.weights.ctypes.data, avg.out.data_ptr(), D.stream()))
        ev[3].record()

    for _ in range(max(3, args.warmup)):
        flush.fill_(1.0)
        one_step()
    barrier()
    # (1) the timed step: the public averaging call (compress -> allgather -> decode,
    #     pipelined in chunk pieces), one CUDA-event pair per step
    step_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    launches0 = F.kernel_launches()
    with ClockSampler(local_rank) as clk:
        barrier()
        for i in range(args.steps):
            flush.fill_(float(i))
            step_ev[i][0].record()
            one_step()
            step_ev[i][1].record()
        barrier()
    launches = F.kernel_launches() - launches0
    avg.check()
    step_ms = np.array([e[0].elapsed_time(e[1]) for e in step_ev])
    # (2) stage breakdown (not pipelined): compress | allgather | decode-average
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for _ in range(2):                          # NCCL communicator set-up stays out of the stage times
        one_step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    barrier()
    for i in range(args.steps):
        flush.fill_(float(i))
        one_step(evs[i])
    barrier()
    st = np.array([[evs[i][0].elapsed_time(evs[i][1]), evs[i][1].elapsed_time(evs[i][2]),
                    evs[i][2].elapsed_time(evs[i][3])] for i in range(args.steps)])
    # (3) the dominant kernel alone for the roofline: the fused compress of the
    #     65536-sample chunks, CUDA events on the stream it is launched on
    kalg = C.c_uint64(0)
    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(float(i))
        kev[i][0].record()
        _lib.check(_lib.lib.fgc_profile_fused_compress(avg.plan.handle, grad.data_ptr(), _lib.DTYPE_F32,
                                                       avg.message.data_ptr(), avg.flags.data_ptr(), D.stream(),
                                                       C.byref(kalg)))
        kev[i][1].record()
    barrier()
    k_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in kev]))
    local = np.array([step_ms.mean(), st[:, 0].mean(), st[:, 1].mean(), st[:, 2].mean(), k_ms])
    if world > 1:
        t = torch.tensor(local, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        local = t.cpu().numpy()
    ms, c_ms, s_ms, d_ms, k_ms = [float(x) for x in local]

    # ---- uncompressed baseline collective: fp32 allreduce of the gradient
    allreduce_ms = None
    if world > 1:
        buf = grad.clone()
        for _ in range(3):
            comm.allreduce_sum_(buf)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            comm.allreduce_sum_(buf)
        e1.record()
        barrier()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        allreduce_ms = float(t.item())

    # ---- end to end through the public API with pinned host buffers
    host_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
    host_in.copy_(grad.cpu())
    host_out = torch.empty(n, dtype=torch.float32, pin_memory=True)

    def e2e_step():
        # the public host-buffer call: its PCIe copies overlap the codec kernels
        avg.step_host(host_in, host_out, wait=False)

    for _ in range(2):
        e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        e2e_step()
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    transport = avg.transport if world > 1 else None
    avg.close()
    if rank != 0:
        return
    hbm, peak_kind = peaks()
    job_bytes = 4.0 * n * world
    value = job_bytes / (ms * 1e-3) / 1e9
    # roofline of the dominant kernel (algorithmic bytes per launch / its time)
    comp_bytes = 4.0 * n + M
    dec_bytes = float(world) * M + 4.0 * n
    dom = ("compress", comp_bytes, c_ms) if c_ms >= d_ms else ("decode_average", dec_bytes, d_ms)
    kernel_name = dom[0]
    if dom[0] == "compress" and kalg.value:
        # the fused compress kernel alone: its own algorithmic bytes over its own time
        dom = ("compress", float(kalg.value), k_ms)
        kernel_name = "k_fused_compress"
    achieved = dom[1] / (dom[2] * 1e-3) / 1e9
    traffic = None        # DRAM bytes per launch of that kernel from the committed ncu --set full capture
    try:
        tr = json.load(open(Path(__file__).resolve().parent / "profiles" / "traffic.json"))
        default_cfg = not args.n and args.theta_drop is None and args.n_bits is None and args.mbits is None
        if default_cfg and (dom[0] == "compress" or world == 1):
            traffic = tr.get(args.workload, {}).get(dom[0])
    except (OSError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic gaussian sigma=1e-2 (torch.randn, seed 1000+rank)",
        "config": workload_config(args, wl, world),
        "sync_ms": ms, "transport": transport,
        "stages_ms": {"compress": c_ms, "allgather": s_ms, "decode_average": d_ms,
                      "note": "unpipelined stage breakdown (NCCL allgather); ms_per_step is the public averaging "
                              "call, whose exchange overlaps the codec kernels"},
        "allreduce_fp32_ms": allreduce_ms,
        "sync_vs_allreduce": (ms / allreduce_ms) if allreduce_ms else None,
        "nvlink": {"bytes_in_per_rank": (world - 1) * M, "bytes_out_per_rank": (world - 1) * M,
                   "achieved_gbs_per_rank": (world - 1) * M / (ms * 1e-3) / 1e9,
                   "peak_gbs": 900.0, "peak_kind": "nominal per direction per GPU",
                   "frac": (world - 1) * M / (ms * 1e-3) / 1e9 / 900.0,
                   "measured_peer_copy_gbs": 770.0,
                   "exchange": {"1": "direct peer reads", "2": "kernel pushes"}.get(
                       os.environ.get("FGC_EXCHANGE_DIRECT", "0")[:1], "copy-engine pushes")
                       if transport == "peer" else transport,
                   "note": "allgather receive (W-1)*M per rank over the step time (capacity bytes: an upper "
                           "bound under direct peer reads, which fetch each segment's used bytes only)"},
        "message_bytes": M, "compression_ratio": 4.0 * n / M,
        "roofline": {"bound": "hbm", "kernel": kernel_name, "achieved": achieved, "peak": hbm, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "algorithmic_bytes": dom[1], "kernel_ms": dom[2],
                     "compress_stage": {"ms": c_ms, "algorithmic_bytes": comp_bytes,
                                        "achieved": comp_bytes / (c_ms * 1e-3) / 1e9},
                     "step_frac": ((comp_bytes + dec_bytes) / ((c_ms + d_ms) * 1e-3) / 1e9) / hbm},
        "e2e": {"value": job_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        gbs, cores, sample = cpu_reference(wl, seconds_budget=15.0)
        line["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample,
                                "host": host_info()}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=sorted(WORKLOADS))
    ap.add_argument("--n", "--n-floats", dest="n", type=int, default=None)
    ap.add_argument("--mode", default="count", choices=["count", "energy"],
                    help="sparsification rule (spectral.py:124-139); the headline is count mode")
    ap.add_argument("--theta-drop", type=float, default=None,
                    help="override the workload's theta (BASELINE config 3 sweeps keep 0.01/0.05/0.1/0.3)")
    ap.add_argument("--n-bits", type=int, default=None, help="override the range-float width (config 4 sweep)")
    ap.add_argument("--mbits", type=int, default=None, help="override the mantissa bits (with --n-bits)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default=None, choices=["peer", "nccl"],
                    help="exchange for N>1: peer-to-peer copies (default) or one NCCL allgather")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.n:
        wl["n"] = args.n
    if args.theta_drop is not None:
        wl["theta"] = args.theta_drop
    if args.n_bits is not None:
        wl["n_bits"] = args.n_bits
        wl["mbits"] = args.mbits if args.mbits is not None else {4: 2, 6: 2, 8: 3, 16: 9}.get(args.n_bits, 3)
    elif args.mbits is not None:
        wl["mbits"] = args.mbits
    wl["mode"] = args.mode
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` outside torchrun: launch the N ranks ourselves
        # (one process per GPU) and pass rank 0's JSON line through
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        # (torch.distributed.run's own parser would take `--n` for an
        # abbreviation of its options: pass it under its long alias)
        fwd = ["--n-floats" + a[3:] if a == "--n" or a.startswith("--n=") else a for a in sys.argv[1:]]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *fwd]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} ranks",
              file=sys.stderr, flush=True)
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, wl, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
