import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running oracle pin (still part of the default suite)")


def pytest_sessionstart(session):
    """Build the CUDA library (sm_100a) and the oracle from THIS source tree before any test runs -- an mtime
    no-op when both are fresh -- so GPU tests never exercise a stale libamr.so."""
    from paper_2508_05020_b200 import build as B
    import oracle
    B.build()
    oracle.build()
