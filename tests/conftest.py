"""Shared test fixtures.  GPU tests are marked ``gpu`` (run on the B200 box);
everything else runs on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")


def small_instance(rng, m, n, family):
    """Small seeded instance of one bound family (test fixture, modelled on the
    reference's nnls / bvls / mixed families, pkg/tests/conftest.py:9-35)."""
    if family == "nnls":
        a = np.abs(rng.standard_normal((m, n))) + 0.05
        y = a @ np.maximum(rng.standard_normal(n), 0.0) + 0.1 * rng.standard_normal(m)
        lo, hi = np.zeros(n), np.full(n, np.inf)
    elif family == "bvls":
        a = rng.standard_normal((m, n))
        y = rng.standard_normal(m)
        b = float(rng.uniform(0.1, 1.5))
        lo, hi = np.full(n, -b), np.full(n, b)
    elif family == "mixed":
        a = np.abs(rng.standard_normal((m, n))) + 0.05
        y = a @ np.maximum(rng.standard_normal(n), 0.0) + 0.1 * rng.standard_normal(m)
        lo, hi = np.zeros(n), np.full(n, np.inf)
        fin = rng.permutation(n)[: n // 2]
        hi[fin] = rng.uniform(0.2, 2.0, fin.size)
    else:
        raise ValueError(family)
    return np.asfortranarray(a), y, lo, hi


def medium_nnls(seed=4242, m=300, n=600, nnz=30):
    """Seeded screened-NNLS instance with a few hundred passive columns at the
    active-set optimum (regenerated instead of stored in the fixtures)."""
    rng = np.random.default_rng(seed)
    a = rng.random((m, n))
    a /= np.linalg.norm(a, axis=0)
    x0 = np.zeros(n)
    x0[rng.permutation(n)[:nnz]] = np.abs(rng.standard_normal(nnz))
    y = a @ x0 + 0.01 * rng.standard_normal(m)
    return np.asfortranarray(a), y, np.zeros(n), np.full(n, np.inf)


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def rng():
    return np.random.default_rng(2024)
