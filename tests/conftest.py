import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the round-end GPU tier)")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


@pytest.fixture(scope="session")
def ctx():
    """One GPU context for the session; the CUDA path must load (no fallback)."""
    from paper_2203_11733_b200._native import Context
    c = Context(0)
    c.set_stream(0)  # torch's (legacy) default stream: device tensors made by the tests are ordered with our work
    yield c
    c.close()
