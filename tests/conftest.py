import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run through gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def built():
    """Builds libqsv.so and the oracle libraries once per session."""
    from paper_2512_18995_b200 import build as b
    from oracle import oracle

    b.build()
    oracle.build()
    return True
