"""Test configuration.

-m "not gpu": oracle vs the reference's golden vectors, host logic, C-ABI exports,
              multi-process (gloo) sharding logic -- runs in the CPU container.
-m gpu:       parity of the CUDA path (through the C ABI) against the oracle and
              the golden fixtures -- runs on a B200.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libtdw.so")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def golden(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def term_scale(P, A, B, C, s, d, dt, power):
    """Magnitude scale of the closed-form terms of one triple: K (s + r_max)^p 2 pi.
    Coefficients that are small because of cancellation are compared against it."""
    L = np.max([np.linalg.norm(P - A, axis=1), np.linalg.norm(P - B, axis=1),
                np.linalg.norm(P - C, axis=1)], axis=0)
    K = 1.0 / (4.0 * np.pi * dt ** d)
    return K * (s + L) ** power * 2.0 * np.pi


def coeff_err(got, ref, scale):
    """max |got - ref| / max(|ref|, term scale)."""
    return float(np.max(np.abs(got - ref) / np.maximum(np.maximum(np.abs(ref), scale), 1e-300)))


def per_step_rel(x, ref):
    """Per-step relative L2 error of a (steps, ns) history against a reference."""
    num = np.linalg.norm(x - ref, axis=1)
    den = np.maximum(np.linalg.norm(ref, axis=1), 1e-300)
    return num / den
