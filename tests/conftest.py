import os
import sys
from pathlib import Path

os.environ.setdefault("HCNN_TEST_MODE", "1")
ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import pytest  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the engine through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(GOLDEN / "golden_small.npz"))


@pytest.fixture(scope="session")
def golden_hashes():
    import json
    return json.loads((GOLDEN / "golden_hashes.json").read_text())


@pytest.fixture()
def rng():
    return np.random.default_rng(12345)
