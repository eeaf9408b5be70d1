"""Time fgc_compress and fgc_decode_average for W stacked messages on one GPU
(what every rank of a W-GPU run decodes).  argv: n  W...  (defaults 25.6M, 1 2 4 8)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, _device as D
from paper_1811_08596_b200.codec import _compress_device

torch.cuda.set_device(0)
import ctypes, os
if os.environ.get("FGC_KNOBS"):
    _lib.lib.fgc_debug_set_fused_knobs(ctypes.c_uint32(int(os.environ["FGC_KNOBS"])))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
Ws = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
msgs = []
for w in range(max(Ws)):
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(w)) * 1e-2
    plan, m, _ = _compress_device(g, _lib.DTYPE_F32, cfg)
    msgs.append(m)
stacked = torch.stack(msgs)
out = torch.empty(n, dtype=torch.float32, device="cuda")
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


flags = torch.zeros(1, dtype=torch.int32, device="cuda")
msg = plan.new_message()
tc = timed(lambda: _lib.check(_lib.lib.fgc_compress(plan.handle, g.data_ptr(), _lib.DTYPE_F32, msg.data_ptr(),
                                                     flags.data_ptr(), D.stream())))
print(f"compress n={n}: {tc:8.1f} us")
for W in Ws:
    w = np.full(W, 1.0 / W)
    t = timed(lambda: _lib.check(_lib.lib.fgc_decode_average(plan.handle, stacked.data_ptr(), W, plan.message_bytes,
                                                             w.ctypes.data, out.data_ptr(), D.stream())))
    print(f"decode W={W}: {t:8.1f} us")
