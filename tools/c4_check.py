"""Quick check of an alternate compress kernel (env ALT: 4 = fused4.cu, 1 =
fused_w.cu) against the default 2-CTA one and the oracle.
argv: n theta nbits mbits"""
import ctypes, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import oracle as O
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, debug

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4 * 65536 + 5402
theta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
nm = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (8, 3)
lib = _lib.lib
lib.fgc_debug_set_compress_kernel.argtypes = [ctypes.c_int]
torch.cuda.set_device(0)
g = (torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(3)) * 1e-2)
q = F.calibrate([g[: min(n, 4 * 65536)].double().cpu().numpy()], *nm)
cfg = F.CodecConfig(F.SparsificationSpec(theta), q)
res = {}
ALT = int(os.environ.get("ALT", "4"))
for k in (2, ALT):
    lib.fgc_debug_set_compress_kernel(k)
    spec = debug.forward_spectrum(g, cfg)
    m = F.compress(g, cfg)
    torch.cuda.synchronize()
    res[k] = (spec, debug.message_bytes(m))
s2, s4 = res[2][0], res[ALT][0]
err = np.abs(s4.astype(np.complex128) - s2.astype(np.complex128)).max() / np.sqrt(np.mean(np.abs(s2.astype(np.complex128)) ** 2))
print("spectrum max |alt - 2| / rms:", err)
# oracle encode of the 4-kernel's coefficients
lat = O.lattice(q.min, q.max, q.n_bits, q.mantissa_bits, q.eps)
lengths = O.chunk_lengths(n, 65536)
layout, total = O.device_layout(n, 65536, theta, nm[0])
buf = res[ALT][1]
pos = 0
bad = 0
for c, L in enumerate(lengths):
    b = L // 2 + 1
    _, ch = O.encode_spectrum(s4[pos:pos + b], L, theta, "count", lat)
    off, bmo, co, _ = layout[c]
    nnz = int.from_bytes(buf[off:off + 4], "little")
    bm = buf[off + bmo: off + bmo + (2 * b + 7) // 8]
    cb = buf[off + co: off + co + (nnz * nm[0] + 7) // 8]
    ok = nnz == ch.codes.size and bm == O.flags_to_bytes(ch.bitmap) and cb == O.codes_to_bytes(ch.codes, nm[0])
    if not ok:
        bad += 1
        if bad < 4:
            print("chunk", c, "differs: nnz", nnz, ch.codes.size, "bm eq", bm == O.flags_to_bytes(ch.bitmap))
    pos += b
print("chunks", len(lengths), "differing", bad, "| msg equal to 2-CTA kernel:", res[2][1] == res[ALT][1])
if res[2][1] != res[ALT][1]:
    a2, aa = np.frombuffer(res[2][1], np.uint8), np.frombuffer(res[ALT][1], np.uint8)
    d = np.nonzero(a2 != aa)[0]
    print("differing bytes", d.size, "first", d[:8])
    for c, (off, bmo, co, _) in enumerate(layout):
        nxt = layout[c + 1][0] if c + 1 < len(layout) else len(a2)
        dd = d[(d >= off) & (d < nxt)]
        if dd.size:
            print(" chunk", c, "seg rel", (dd[:6] - off).tolist(), "bitmap at", bmo, "codes at", co, "seg len", nxt - off)
            break
