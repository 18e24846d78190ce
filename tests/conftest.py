import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible (no CPU fallback exists)")
    return 0


def history_err(h, ref) -> float:
    """Max elementwise difference of two relative-residual histories, relative to
    max(ref, 1e-6): relative for the entries that carry information, absolute (scaled)
    for entries already at round-off level. Parity target (BASELINE.json): <= 1e-10."""
    h, ref = np.asarray(h, dtype=float), np.asarray(ref, dtype=float)
    n = min(h.size, ref.size)
    return float(np.max(np.abs(h[:n] - ref[:n]) / np.maximum(ref[:n], 1e-6)))
