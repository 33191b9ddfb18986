"""Test configuration: the `gpu` marker (tests that need a B200) and repo-root imports.

`-m "not gpu"` runs the oracle-vs-reference pinning, the golden fixtures, the C-ABI
export check and the multi-process (gloo) shard logic on CPU. `-m gpu` runs the parity
tests proper: CUDA kernels through the C-ABI against the oracle and the fixtures.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import C_Oracle
    return C_Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, REF_DIR
    if not (REF_DIR / "libkvq_ref.so").exists():
        try:
            from oracle.oracle import build
            build()
        except Exception:
            pass
    if not (REF_DIR / "libkvq_ref.so").exists():
        pytest.skip("reference shim not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def kvq():
    from paper_2502_14882_b200 import kvq as k
    if not k.device_available():
        pytest.fail("no CUDA device: gpu tests must run on a B200 (no CPU fallback exists)")
    return k


@pytest.fixture(scope="session")
def kvq_host():
    """The product library without requiring a device: host-side paths only (argument and
    file-format validation, which run before any device work)."""
    from paper_2502_14882_b200 import kvq as k
    k.lib()
    return k
