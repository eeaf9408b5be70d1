"""A/B of the fused compress pack for 8-bit codes: direct byte stores into the
message (default) vs the shared-memory staged stream (knob 32); checks the
messages are byte-equal and times fgc_compress at 25.6M floats."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, _device as D, debug
from paper_1811_08596_b200.codec import _compress_device
n = 25_600_000
g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
_lib.lib.fgc_debug_set_fused_knobs.argtypes = [ctypes.c_uint32]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
res = {}
for knob in (32, 0, 32, 0):
    _lib.lib.fgc_debug_set_fused_knobs(knob)
    plan, msg, flags = _compress_device(g, _lib.DTYPE_F32, cfg)
    torch.cuda.synchronize()
    b = msg.cpu().numpy().tobytes()
    ts = []
    for _ in range(10):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(_lib.lib.fgc_compress(plan.handle, g.data_ptr(), _lib.DTYPE_F32, msg.data_ptr(), flags.data_ptr(), D.stream()))
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    res.setdefault(knob, []).append(b)
    print("knob", knob, "compress us", round(float(np.median(ts)), 1))
print("messages equal:", res[0][0] == res[32][0] == res[0][1] == res[32][1])
