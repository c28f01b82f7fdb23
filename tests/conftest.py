"""Test configuration: `gpu` marker for tests that need a B200 (run with -m gpu)."""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = os.environ.get("PPMOE_REFERENCE_SRC", "/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def reference_available() -> bool:
    return Path(REFERENCE_SRC, "moebal", "__init__.py").exists()


def import_reference():
    """The unmodified reference package, only in the build container."""
    if not reference_available():
        pytest.skip("reference sources not present (GPU box): goldens cover this")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import moebal

    return moebal


@pytest.fixture
def rng():
    import numpy as np

    return np.random.default_rng(20240817)
