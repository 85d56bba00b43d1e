"""Test configuration.

Markers: `gpu` = needs a B200 (run with `-m gpu` on the GPU box); everything
else runs on CPU (`-m "not gpu"`). GPU tests do not skip when CUDA is absent:
they fail, so a missing device can never pass silently.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(autouse=True)
def _retune_after_env_changes():
    """The library reads its WF_* tuning variables once; tests that
    monkeypatch them call _native.reload_tuning(), and this fixture (set up
    before, torn down after monkeypatch) re-reads the restored environment."""
    yield
    from paper_1803_00737_b200 import _native

    _native.reload_tuning()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")


class Golden:
    """Lazy view over tests/golden/*.npz (reference-generated vectors)."""

    def __init__(self, name):
        self._z = np.load(GOLDEN / f"{name}.npz")

    def __getitem__(self, key):
        return self._z[key]

    def __contains__(self, key):
        return key in self._z.files

    def keys(self):
        return self._z.files


@pytest.fixture(scope="session")
def golden_fusion():
    return Golden("fusion")


@pytest.fixture(scope="session")
def golden_transforms():
    return Golden("transforms")


@pytest.fixture(scope="session")
def golden_metrics():
    return Golden("metrics")


@pytest.fixture(scope="session")
def golden_pnm():
    return Golden("pnm")
