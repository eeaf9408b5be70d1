"""Timeline of the host-buffer averaging step (fgc_average_host) at one rank:
when each H2D piece, each piece's decode and each D2H piece completes
(FGC_EXCHANGE_TRACE=1 events), in ms from the step start.  argv: pieces"""
import ctypes
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["FGC_EXCHANGE_TRACE"] = "1"
if len(sys.argv) > 1:
    os.environ["FGC_HOST_PIECES"] = sys.argv[1]
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib
from paper_1811_08596_b200.comm import GradientAverager

n = 25_600_000
hin = torch.randn(n).mul_(1e-2).pin_memory()
hout = torch.empty(n, pin_memory=True)
q = F.calibrate([hin[:1 << 20].numpy()], 8, 3)
avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0])
lib = _lib.lib
lib.fgc_debug_exchange_trace.argtypes = [ctypes.c_char_p, ctypes.c_int]
buf = ctypes.create_string_buffer(1 << 16)
for it in range(4):
    torch.cuda.synchronize()
    avg.step_host(hin, hout, wait=True)
    lib.fgc_debug_exchange_trace(buf, len(buf))
lines = buf.value.decode().strip().splitlines()
print(" | ".join(f"{l.split()[0]} {float(l.split()[1]):.3f}" for l in lines))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
os.environ.pop("FGC_EXCHANGE_TRACE")
# back-to-back steps queued without waiting (argv[2] = K): the cross-step
# overlap of one step's copy-out with the next step's copy-in
if len(sys.argv) > 2:
    K = int(sys.argv[2])
    os.environ["FGC_EXCHANGE_TRACE"] = "1"
    torch.cuda.synchronize()
    lib.fgc_debug_exchange_trace(buf, len(buf))          # clear
    for it in range(K):
        avg.step_host(hin, hout, wait=False)
    torch.cuda.synchronize()
    lib.fgc_debug_exchange_trace(buf, len(buf))
    lines = buf.value.decode().strip().splitlines()
    print(f"{K} back-to-back steps:")
    print(" | ".join(f"{l.split()[0]} {float(l.split()[1]):.3f}" for l in lines))
