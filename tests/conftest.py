"""pytest configuration: the `gpu` marker, shared fixtures, golden loader.

`-m "not gpu"` (the CPU box): oracle pins, host-side logic, C-ABI load/export
checks, world_size-2 gloo tests.  `-m gpu` (a B200 box): CUDA-vs-oracle
parity through the C-ABI.
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) GPU; parity through the C-ABI")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (run under gpurun --gpus N)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle
