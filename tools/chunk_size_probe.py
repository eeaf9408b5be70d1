"""Compress / decode_average time of a 25.6M-float gradient at chunk sizes
other than 65536 (the generic path: batched DFT engine + per-chunk select +
pack).  argv: n chunk..."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, _device as D
from paper_1811_08596_b200.codec import _compress_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
chunks = [int(x) for x in sys.argv[2:]] or [4096, 16384, 65536]
g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
q = F.tune_eps(-200.0, 200.0, 8, 3)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for chunk in chunks:
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q, chunk_size=chunk)
    plan, msg, flags = _compress_device(g, _lib.DTYPE_F32, cfg)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    w = np.ones(1)
    tc = timed(lambda: _lib.check(_lib.lib.fgc_compress(plan.handle, g.data_ptr(), _lib.DTYPE_F32, msg.data_ptr(),
                                                        flags.data_ptr(), D.stream())))
    td = timed(lambda: _lib.check(_lib.lib.fgc_decode_average(plan.handle, msg.data_ptr(), 1, plan.message_bytes,
                                                              w.ctypes.data, out.data_ptr(), D.stream())))
    print(f"chunk {chunk:6d}: compress {tc:8.1f} us  decode {td:8.1f} us  ({4 * n / (tc + td) / 1e3:.0f} GB/s)")
