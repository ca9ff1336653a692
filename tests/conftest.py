import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

# the library's COVGPU_* switches (engine forcing for the parity tests) are
# honoured only under this flag (csrc/covgpu.cu hook_env)
os.environ.setdefault("COVGPU_TEST_HOOKS", "1")

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libcovgpu.so")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN / "golden.npz"))


@pytest.fixture(scope="session")
def golden_cfg5():
    return dict(np.load(GOLDEN / "golden_cfg5.npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1303_2285_b200 import _native

    _native.lib()  # fail loudly if the extension is missing on a GPU box
    return torch.device("cuda", 0)
