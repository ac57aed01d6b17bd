"""Builds tests/cpp/dropin_test.cpp (reference-style C++ tests) against the
C++ drop-in header include/specden/specden_b200.hpp and runs it on the GPU."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_cpp_dropin_binary(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2505_11564_b200 import build
    lib = build.build()
    exe = tmp_path / "dropin_test"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'shims'}",
           "-I/usr/local/cuda/include", str(ROOT / "tests" / "cpp" / "dropin_test.cpp"), str(lib),
           f"-Wl,-rpath,{lib.parent}", "-L/usr/local/cuda/lib64", "-lcudart", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-1500:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "0 failed" in r.stdout
