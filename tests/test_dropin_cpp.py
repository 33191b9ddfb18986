"""The C++ drop-in headers (include/kvq/*.hpp): they compile against the C-ABI with the
reference's flags (CPU), and the reference's known-answer tests pass through them on the
GPU (tests/cpp/test_dropin.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_2502_14882_b200"


def build_binary(tmp_path: Path) -> Path:
    exe = tmp_path / "test_dropin"
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
           str(ROOT / "tests" / "cpp" / "test_dropin.cpp"), f"-L{LIBDIR}", "-lkvq_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_dropin_headers_compile(tmp_path):
    build_binary(tmp_path)


@pytest.mark.gpu
def test_dropin_reference_known_answers(tmp_path):
    exe = build_binary(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "all passed" in res.stdout
