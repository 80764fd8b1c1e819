import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity of the CUDA path vs the oracle")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (run under gpurun --gpus N)")
    config.addinivalue_line("markers", "slow: long-running oracle check")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:  # pragma: no cover
        ngpu = 0
    for it in items:
        if "multigpu" in it.keywords and ngpu < 2:
            it.add_marker(pytest.mark.skip(reason="needs >= 2 GPUs"))
