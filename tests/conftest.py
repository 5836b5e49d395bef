"""Test configuration.

Markers: `gpu` tests need a B200 (they call the sm_100a library); everything
else runs on CPU.  The oracle (oracle/, TEST INFRASTRUCTURE) is the checker.
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a library)")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        p = GOLDEN / name
        return json.loads(p.read_text()) if p.suffix == ".json" else np.load(p)
    return load


@pytest.fixture(scope="session")
def oracle():
    from oracle import zo2_oracle
    zo2_oracle.lib()
    return zo2_oracle


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    torch.cuda.init()
    return torch.device("cuda:0")
