"""Minimal decode check for one size: compress + decompress vs oracle."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1811_08596_b200 as F
import oracle as O
n = int(sys.argv[1])
rng = np.random.default_rng(7)
g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
q = F.calibrate([g], 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
msg = F.compress(g, cfg)
ref = O.decompress(O.from_wire(F.serialize(msg)))
try:
    got = F.decompress(msg)
    print(n, "rel", np.linalg.norm(got - ref) / np.linalg.norm(ref))
except Exception as e:
    print(n, "ERR", str(e)[:200])
