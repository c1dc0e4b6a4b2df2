"""Shared test setup.

Markers: `gpu` tests need a CUDA device (the B200 parity gate); everything
else runs on CPU. The oracle (C restatement, oracle/ezq_oracle.c) is test
infrastructure and is built on demand; the engine library is built by
__graft_entry__.build() (and on demand here when a GPU box lacks it).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200 parity gate)")


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def ensure_engine():
    from paper_2403_02775_b200 import native
    if not os.path.exists(native.LIB_PATH):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2403_02775_b200", "csrc")],
                       check=True)
    return native


@pytest.fixture(scope="session")
def N():
    """The engine (ctypes binding of libezq_b200.so)."""
    return ensure_engine()


@pytest.fixture(scope="session")
def O():
    """The oracle (C restatement) -- checker only."""
    from oracle import pyoracle
    pyoracle.build()
    return pyoracle


@pytest.fixture(scope="session")
def gpu(N):
    if not _cuda_available():
        pytest.skip("no CUDA device")
    return N


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_cfg(arr):
    from paper_2403_02775_b200.native import Config
    a = [float(v) for v in arr]
    return Config(bits=int(a[0]), sigma_n=a[1], lr=a[2], beta1=a[3], beta2=a[4], eps=a[5],
                  steps=int(a[6]), select="fixed" if int(a[7]) else "best", select_step=int(a[8]))


def golden_quant_files():
    return sorted(f for f in os.listdir(GOLDEN) if f.startswith("quant_"))
