import gzip
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(HERE, "golden")

# The per-rule kernel compiler (csrc/wcoj_jit.cu) is off for the bulk of the
# suite: hundreds of small golden programs would each schedule NVRTC builds
# that finish after their test. tests/test_gpu_jit.py and the BASELINE-size
# parity tests turn it on (fixture `jit`) and compare both kernel families.
os.environ.setdefault("SRDL_JIT", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsrdl.so")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rb") as fh:
            return json.loads(fh.read())
    with open(path, "rb") as fh:
        return json.loads(fh.read())


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture
def jit():
    """Per-rule kernels on, compiled on first use (synchronously)."""
    from paper_2604_20073_b200 import device as dev

    prev = dev.jit_mode("sync")
    try:
        yield dev
    finally:
        dev.jit_mode(prev)


@pytest.fixture
def audited():
    """Enable the execution audit (reference test mode) for one test."""
    from paper_2604_20073_b200 import audit

    before = audit.enabled
    audit.enabled = True
    audit.reset()
    try:
        yield audit
    finally:
        audit.enabled = before
        audit.reset()
