import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpygs.so")
    config.addinivalue_line("markers", "slow: full-size workloads (minutes)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _refresh_library_knobs(monkeypatch):
    """libpygs reads its PYG_* tuning knobs once; tests that monkeypatch them get them re-read
    (monkeypatch.setenv wrapped) and restored after the test."""
    mod = sys.modules.get("paper_1903_02428_b200._abi")
    orig = monkeypatch.setenv

    def setenv(name, value, prepend=None):
        orig(name, value, prepend)
        m = sys.modules.get("paper_1903_02428_b200._abi")
        if m is not None and name.startswith("PYG_"):
            m.lib.pyg_refresh_env()

    monkeypatch.setenv = setenv
    yield
    monkeypatch.undo()
    m = sys.modules.get("paper_1903_02428_b200._abi") or mod
    if m is not None:
        m.lib.pyg_refresh_env()
