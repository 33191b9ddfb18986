"""C-ABI boundary checks that need no GPU: the product library loads, exports exactly
the entry points include/kvq_capi.h declares, is not linked against the oracle, and
refuses to compute without a device (no CPU fallback)."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2502_14882_b200" / "libkvq_b200.so"


def declared_symbols():
    text = (ROOT / "include" / "kvq_capi.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kvq_[a-z0-9_]+)\s*\(", text)))


def exported_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_library_built():
    assert LIB.exists(), "run __graft_entry__.build() first"


def test_every_declared_symbol_is_exported():
    decl = declared_symbols()
    assert len(decl) >= 30
    missing = [s for s in decl if s not in exported_symbols()]
    assert not missing, missing


def test_product_library_does_not_link_oracle():
    deps = subprocess.run(["ldd", str(LIB)], capture_output=True, text=True).stdout
    assert "kvq_ref" not in deps and "kvq_oracle" not in deps
    syms = exported_symbols()
    assert not any(s.startswith(("kvqo_", "kvqr_")) for s in syms)


def test_python_binding_loads_every_symbol():
    from paper_2502_14882_b200 import kvq
    L = kvq.lib()
    for s in declared_symbols():
        assert hasattr(L, s)


def test_no_cpu_fallback_without_device():
    from paper_2502_14882_b200 import kvq
    if kvq.device_available():
        pytest.skip("a GPU is present")
    with pytest.raises(kvq.CudaError):
        kvq.pack(np.array([1, 0, 1], np.uint32), 1)
    with pytest.raises(kvq.CudaError):
        kvq.compute_stats(np.ones((2, 2), np.float32))
    with pytest.raises(kvq.CudaError):
        kvq.HybridKVCache.build([np.ones((4, 8), np.float32)], [np.ones((4, 8), np.float32)],
                                kvq.QuantizationConfig(1), kvq.CalibrationParams())


def test_config_errors_precede_device_check():
    """Argument validation mirrors the reference's exception classes even off-GPU."""
    from paper_2502_14882_b200 import kvq
    with pytest.raises(kvq.ConfigError):
        kvq.pack(np.array([1], np.uint32), 3, 8)  # bitpack.hpp:145-148
    with pytest.raises(kvq.ConfigError):
        kvq.pack(np.array([1], np.uint32), 1, 12)
    with pytest.raises(kvq.ConfigError):
        kvq.KernelConfig(0, 1, 1).validate()  # kernels.hpp:35-39
    with pytest.raises(kvq.DomainError):
        kvq.compute_stats(np.zeros((0, 3), np.float32))  # quantize.hpp:65
