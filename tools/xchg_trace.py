"""Timeline of one peer-exchange averaging step (FGC_EXCHANGE_TRACE=1), per rank.  torchrun."""
import ctypes
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["FGC_EXCHANGE_TRACE"] = "1"
import numpy as np
import torch
import torch.distributed as dist
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib
from paper_1811_08596_b200.comm import GradientAverager, NcclComm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl")
n = 25_600_000
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(rank)) * 1e-2
avg = GradientAverager(n, cfg, np.full(world, 1.0 / world), NcclComm(), transport="peer")
lib = _lib.lib
lib.fgc_debug_exchange_trace.argtypes = [ctypes.c_char_p, ctypes.c_int]
buf = ctypes.create_string_buffer(1 << 16)
for it in range(4):
    dist.barrier()
    torch.cuda.synchronize()
    avg.step(g)
    torch.cuda.synchronize()
    lib.fgc_debug_exchange_trace(buf, len(buf))
    if it == 3:
        lines = buf.value.decode().strip().splitlines()
        print(f"rank {rank}: " + " | ".join(f"{l.split()[0]} {float(l.split()[1]) * 1e3:.0f}" for l in lines), flush=True)
avg.close()
dist.destroy_process_group()
