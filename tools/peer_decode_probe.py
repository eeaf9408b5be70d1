"""Cost of decoding messages that live in a peer GPU's memory (direct peer
reads over NVLink) vs local ones: fgc_decode_average on cuda:0 with the
stacked messages on cuda:1 (peer access enabled) or on cuda:0.
argv: n W (defaults 25.6M, 2)"""
import ctypes
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, _device as D
from paper_1811_08596_b200.codec import _compress_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.cuda.set_device(0)
import os
if os.environ.get("FGC_KNOBS"):
    _lib.lib.fgc_debug_set_fused_knobs(ctypes.c_uint32(int(os.environ["FGC_KNOBS"])))
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
msgs = []
for w in range(W):
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(w)) * 1e-2
    plan, m, _ = _compress_device(g, _lib.DTYPE_F32, cfg)
    msgs.append(m)
local = torch.stack(msgs)
remote = local.to("cuda:1")
torch.cuda.synchronize(1)
print("peer access 0->1:", torch.cuda.can_device_access_peer(0, 1))
# enable peer access from device 0 to device 1 (torch does it lazily for copies; do it explicitly)
import cuda.bindings.runtime as cr  # cuda-python
cr.cudaSetDevice(0)
print("enable peer:", cr.cudaDeviceEnablePeerAccess(1, 0))
out = torch.empty(n, dtype=torch.float32, device="cuda:0")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
w = np.full(W, 1.0 / W)


def timed(src, reps=10):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(_lib.lib.fgc_decode_average(plan.handle, src.data_ptr(), W, plan.message_bytes, w.ctypes.data,
                                               out.data_ptr(), D.stream()))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts)), out.clone()


tl, ol = timed(local)
tr, orr = timed(remote)
print(f"decode W={W} local {tl:.1f} us, remote (peer) {tr:.1f} us, equal: {torch.equal(ol, orr)}")
