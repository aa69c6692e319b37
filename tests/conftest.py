import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libmerbit_b200.so")
    config.addinivalue_line("markers", "slow: large-scale case (R-MAT scale >= 20)")


@pytest.fixture(scope="session", params=[1, 0], ids=["slots", "staged"])
def ctx(request):
    """A device context per K2 data layout: 1 = lane-major slot copy
    (default), 0 = CSR order staged through shared memory.  Every GPU parity
    test runs under both."""
    import paper_2605_07391_b200 as mb
    c = mb.Context(0)
    c.set_layout(request.param)
    return c


@pytest.fixture(scope="session")
def golden():
    import json
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return {name: json.load(open(os.path.join(here, f"{name}.json")))
            for name in ("walkthrough", "fuzz_corpus", "pagerank")}


def gpu_shared_between_processes() -> bool:
    """False when device 0 is in an exclusive compute mode (a second process
    could not create a context): the multi-process tests then skip."""
    try:
        import pynvml
        pynvml.nvmlInit()
        try:
            mode = pynvml.nvmlDeviceGetComputeMode(pynvml.nvmlDeviceGetHandleByIndex(0))
        finally:
            pynvml.nvmlShutdown()
        return mode == pynvml.NVML_COMPUTEMODE_DEFAULT
    except Exception:
        return True
