"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/specden_b200.h declares, and its host-side
bookkeeping (layout, partial shapes, rank-ordered combine, tridiagonal
eigensolve, density) matches the oracle / reference semantics."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def sd():
    from paper_2505_11564_b200 import build
    build.build()
    import paper_2505_11564_b200 as sd
    return sd


def declared_symbols():
    hdr = (ROOT / "include" / "specden_b200.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    types = {"sd_status", "sd_stream", "sd_comm", "sd_operator", "sd_lanczos", "sd_apply_fn"}
    return sorted(set(re.findall(r"\b(sd_[a-z0-9_]+)\s*\(", hdr)) - types)


def test_library_exports_every_declared_symbol(sd):
    lib = ROOT / "paper_2505_11564_b200" / "libspecden_b200.so"
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (sd_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert len(declared_symbols()) >= 40


def test_library_targets_sm100a(sd):
    lib = ROOT / "paper_2505_11564_b200" / "libspecden_b200.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_layout_matches_oracle(sd, oracle):
    for dim in (1, 2, 7, 10, 1000, 124439808):
        for n in (1, 2, 3, 4, 8, 16):
            got = [tuple(r) for r in sd.split_evenly(dim, n).shard_bounds]
            assert got == oracle.split_evenly(dim, n)
    l = sd.ShardLayout(10, ((0, 4), (5, 10)))
    with pytest.raises(sd.LayoutError):
        sd.validate_layout(l)
    l = sd.ShardLayout(10, ((0, 3), (3, 6), (6, 8), (8, 10)))
    assert [l.owner(i) for i in range(10)] == [0, 0, 0, 1, 1, 1, 2, 2, 3, 3]
    with pytest.raises(sd.ArgumentError):
        l.owner(10)


def test_host_combine_matches_oracle(sd, oracle):
    import ctypes as C
    from paper_2505_11564_b200 import _lib
    P = 70001
    a = oracle.gaussian_fill(3, 0, P)
    b = oracle.gaussian_fill(4, 0, P)
    ref = oracle.dot(a, b)
    for n in (1, 2, 3, 7, 8):
        rs = oracle.split_evenly(P, n)
        parts = [np.concatenate(oracle.dot_partial(s, e, P, a[s:e], b[s:e])) for s, e in rs]
        for (s, e), p in zip(rs, parts):
            h, sm, t = C.c_uint64(), C.c_uint64(), C.c_uint64()
            _lib.check(_lib.lib().sd_partial_shape(s, e, P, C.byref(h), C.byref(sm), C.byref(t)))
            assert h.value + sm.value + t.value == p.size
        ptrs = (_lib.dp * n)(*[p.ctypes.data_as(_lib.dp) for p in parts])
        out = C.c_double()
        bb = (C.c_uint64 * n)(*[r[0] for r in rs])
        ee = (C.c_uint64 * n)(*[r[1] for r in rs])
        _lib.check(_lib.lib().sd_combine_partials_host(n, bb, ee, P, ptrs, C.byref(out)))
        assert np.float64(out.value).view(np.int64) == np.float64(ref).view(np.int64)
    # out-of-order partials are a protocol error (reduction.hpp:93-94)
    rs = oracle.split_evenly(P, 2)
    parts = [np.concatenate(oracle.dot_partial(s, e, P, a[s:e], b[s:e])) for s, e in rs][::-1]
    ptrs = (_lib.dp * 2)(*[p.ctypes.data_as(_lib.dp) for p in parts])
    bb = (C.c_uint64 * 2)(rs[1][0], rs[0][0])
    ee = (C.c_uint64 * 2)(rs[1][1], rs[0][1])
    with pytest.raises(sd.ProtocolError):
        _lib.check(_lib.lib().sd_combine_partials_host(2, bb, ee, P, ptrs, C.byref(C.c_double())))


def test_rng_and_dense_builders_match_reference(sd, oracle):
    from paper_2505_11564_b200 import _lib
    L = _lib.lib()
    for s, c in ((42, 0), (7, 5), (2 ** 63, 2 ** 40)):
        assert L.sd_keyed_counter(s, c) == oracle.keyed_counter(s, c)
    assert [L.sd_rademacher(7, i) for i in range(16)] == [oracle.rademacher(7, i) for i in range(16)]
    assert np.array_equal(sd.wigner_dense(257, 1.5, 7), oracle.wigner(257, 1.5, 7))
    assert np.array_equal(sd.spiked_dense(200, 1.0, [25.0, -3.0], 1), oracle.spiked(200, 1.0, [25.0, -3.0], 1))
    with pytest.raises(sd.ArgumentError):
        sd.wigner_dense(4096, 1.0, 0)


def test_quadrature_known_answers(sd, oracle):
    r = sd.ritz_decompose([3.5], [])
    assert r.values[0] == 3.5 and r.weights[0] == 1.0
    r = sd.ritz_decompose([0.0, 0.0], [1.0])
    assert np.allclose(r.values, [-1, 1], atol=1e-15) and np.allclose(r.weights, [0.5, 0.5], atol=1e-15)
    d = sd.smooth_density(sd.RitzSpectrum(np.array([0.0]), np.array([1.0])), 1.0, 1001)
    assert abs(d.density[500] - 1 / np.sqrt(2 * np.pi)) < 1e-15
    with pytest.raises(sd.NumericalError):
        sd.ritz_decompose([1.0, float("nan")], [1.0])
    # against the independent Jacobi solver of the oracle on a k=60 Lanczos tridiagonal
    A = oracle.spiked(256, 1.0, [30.0], 3)
    lr = oracle.lanczos_dense(A, 60, reorth=True)
    mine = sd.ritz_decompose(lr["alphas"], lr["betas"])
    v, w = oracle.ritz(lr["alphas"], lr["betas"])
    assert np.max(np.abs(mine.values - v)) <= 1e-11 * np.max(np.abs(v))
    assert np.max(np.abs(mine.weights - w)) <= 1e-12
    assert mine.residual <= 1e-12 and abs(mine.weights.sum() - 1) <= 1e-12
    avg = sd.average_spectra([mine, mine])
    assert np.allclose(np.unique(avg.values), np.unique(mine.values)) and abs(avg.weights.sum() - 1) < 1e-12


def test_columnar_loader(tmp_path):
    # SPEC.md:227 columnar batches: features then target, whitespace separated
    from paper_2505_11564_b200 import mlp
    from paper_2505_11564_b200._lib import ConfigError
    p = tmp_path / "b.txt"
    p.write_text("# x0 x1 y\n1 2 3\n4.5 -1 0.25\n\n")
    x, y = mlp.load_columnar(str(p))
    assert x.tolist() == [[1, 2], [4.5, -1]] and y.tolist() == [[3], [0.25]]
    p.write_text("1 2 3\n4 5\n")
    with pytest.raises(ConfigError):
        mlp.load_columnar(str(p))


def test_cpp_dropin_header_compiles():
    # the C++ drop-in layer (reference names, exception types, hvp/batched_hvp)
    # and the reference-style C++ tests compile on the CPU box; they run on the GPU
    import shutil
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", f"-I{root / 'include'}",
           f"-I{root / 'oracle' / 'shims'}", "-I/usr/local/cuda/include", str(root / "tests" / "cpp" / "dropin_test.cpp")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
