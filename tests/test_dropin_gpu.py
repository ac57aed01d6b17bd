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


SUITES = {"test_sharded_core": 22, "test_runtime": 10, "test_operators": 13}


@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suites_unchanged_against_dropin(suite):
    """The reference's own doctest suites (proj/tests/*.cpp), compiled
    unchanged against the drop-in headers include/specden/*.hpp and linked
    only with libspecden_b200.so (oracle/build_dropin_tests.sh), pass on the
    B200: WorkerPool threads/mailboxes/counters/jitter (pool.hpp:47-94),
    device-resident shards, bitwise layout invariance of probes, dots, axpy,
    scale and dense apply, the error taxonomy, load_dense."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    exe = ROOT / "oracle" / "_ref" / "dropin" / suite
    if not exe.exists():
        pytest.skip("drop-in suites not built (oracle/build_dropin_tests.sh needs the reference tree)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900, cwd=str(exe.parent))
    print(r.stdout[-1500:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert f"test cases: {SUITES[suite]}" in r.stdout, r.stdout[-500:]
