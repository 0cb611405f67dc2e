"""Shared test setup.

Markers: ``gpu`` tests need a CUDA device (B200) and exercise the product through its
C ABI; everything else runs on CPU (oracle vs golden fixtures / live reference, host
control plane, C-ABI symbol checks, gloo multi-process logic).  The CUDA library is
built in-tree on first use (nvcc cross-compiles without a GPU).
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"

import __graft_entry__  # noqa: E402

__graft_entry__.build()


# the vendored reference suite runs in its own pytest process (tests/test_ref_suite.py)
collect_ignore_glob = ["ref_suite/*"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def reference():
    """The real reference package (read-only), when mounted; tests using it are the
    live cross-checks of the oracle and are skipped on the GPU box."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference not mounted")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import kvmix.attention
    import kvmix.pool
    import kvmix.quant
    return kvmix


@pytest.fixture
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def rand_kv(seed, L, N, H, d, dtype=np.float32):
    """K with per-(head, channel) log-uniform [0.5, 4] scales (capture.py:108-112), V ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    k = (rng.standard_normal((L, N, H, d)) * np.exp(rng.uniform(np.log(0.5), np.log(4.0), (H, d))))
    v = rng.standard_normal((L, N, H, d))
    return k.astype(dtype), v.astype(dtype)
