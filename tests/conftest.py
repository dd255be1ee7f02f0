import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

try:
    import hypothesis

    hypothesis.settings.register_profile("mpx", deadline=None, derandomize=True)
    hypothesis.settings.load_profile("mpx")
except ImportError:  # pragma: no cover
    pass

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN / "mpstep_golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_03312_b200 import _native

    _native.load()
    return torch.device("cuda", 0)
