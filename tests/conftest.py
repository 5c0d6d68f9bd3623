import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
# Emulated groups with real barriers put every rank's streams (own + the
# scheduler's two comm streams) in one CUDA context; with the default 8
# hardware work queues, streams alias and a spinning barrier kernel could
# stall an unrelated stream behind it. Must be set before CUDA initialises.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ... and with lazy module loading, the first launch of a kernel may need a
# context synchronisation, which waits for a rank's barrier kernel spinning
# on a peer whose work the (blocked) host thread has not issued yet: load
# every kernel up front instead (CUDA lazy-loading guidance for kernels that
# wait on each other).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def _ensure_built():
    from paper_2311_00257_b200 import build
    if not build.LIB.exists() or not build.ORACLE_LIB.exists() or os.environ.get("AMSP_REBUILD"):
        build.build_library()
        build.build_oracle()


_ensure_built()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
