import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.dirname(__file__)):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libstlg.so")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def import_reference():
    """The unmodified reference package for the engine-hook tests: baseline/_ref (the
    offline install that travels to the GPU box) or, in the dev container, the
    reference tree.  Skips the test when neither is present."""
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "stlmask")):
            if path not in sys.path:
                sys.path.append(path)
            break
    return pytest.importorskip("stlmask")
