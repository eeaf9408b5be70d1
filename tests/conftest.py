import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    here = ROOT / "tests" / "golden"
    meta = json.loads((here / "golden.json").read_text())
    arrays = dict(np.load(here / "golden.npz"))
    return meta, arrays
