"""Compress / decode stage times (CUDA events, L2 flushed) with and without the generic tail chunk."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, _device as D
from paper_1811_08596_b200.comm import GradientAverager

torch.cuda.set_device(0)
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for n in [int(x) for x in sys.argv[1:]] or [390 * 65536, 25_600_000, 40960]:
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
    avg = GradientAverager(n, cfg, [1.0])
    M = avg.plan.message_bytes
    res = []
    for it in range(25):
        flush.fill_(float(it))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        _lib.check(_lib.lib.fgc_compress(avg.plan.handle, g.data_ptr(), _lib.DTYPE_F32, avg.message.data_ptr(),
                                         avg.flags.data_ptr(), D.stream()))
        ev[1].record()
        _lib.check(_lib.lib.fgc_decode_average(avg.plan.handle, avg.message.data_ptr(), 1, M,
                                               avg.weights.ctypes.data, avg.out.data_ptr(), D.stream()))
        ev[2].record()
        torch.cuda.synchronize()
        if it >= 5:
            res.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
    r = np.median(np.array(res), axis=0) * 1e3
    print(f"n={n:>10d} compress {r[0]:7.1f} us  decode {r[1]:7.1f} us", flush=True)
