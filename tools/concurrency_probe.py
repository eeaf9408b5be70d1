"""Fused compress of 390 chunks on one stream, a tail-chunk compress on a
high-priority stream at the same time: who waits for whom."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib
from paper_1811_08596_b200.comm import GradientAverager

torch.cuda.set_device(0)
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
big, small = 390 * 65536, int(sys.argv[1]) if len(sys.argv) > 1 else 40960
gb = torch.randn(big, device="cuda") * 1e-2
gs = torch.randn(small, device="cuda") * 1e-2
A = GradientAverager(big, cfg, [1.0])
Bv = GradientAverager(small, cfg, [1.0])
hi = torch.cuda.Stream(priority=-5)
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def comp(avg, g, stream):
    _lib.check(_lib.lib.fgc_compress(avg.plan.handle, g.data_ptr(), _lib.DTYPE_F32, avg.message.data_ptr(),
                                     avg.flags.data_ptr(), stream.cuda_stream))


res = {"alone_big": [], "alone_small": [], "both_big": [], "both_small": []}
main = torch.cuda.current_stream()
for it in range(25):
    for mode in ("alone_big", "alone_small", "both"):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if mode in ("alone_big", "both"):
            e[0].record(main)
            comp(A, gb, main)
            e[1].record(main)
        if mode in ("alone_small", "both"):
            e[2].record(hi)
            comp(Bv, gs, hi)
            e[3].record(hi)
        torch.cuda.synchronize()
        if it < 5:
            continue
        if mode == "alone_big":
            res["alone_big"].append(e[0].elapsed_time(e[1]))
        elif mode == "alone_small":
            res["alone_small"].append(e[2].elapsed_time(e[3]))
        else:
            res["both_big"].append(e[0].elapsed_time(e[1]))
            res["both_small"].append(e[0].elapsed_time(e[3]))
for k, v in res.items():
    print(f"{k:12s} {np.median(v) * 1e3:8.1f} us")
