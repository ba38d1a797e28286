import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large inputs")


def pytest_sessionstart(session):
    # build the CUDA library (nvcc cross-compiles without a GPU) and the oracle
    from paper_2410_22697_b200 import build
    from oracle import oracle
    build.build()
    oracle.build()
