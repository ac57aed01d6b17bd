"""Parity of the CUDA vector algebra and the device Lanczos engine against the
committed reference fixtures and the oracle. Integer/byte work, every
reference f64 fold and the Gaussian probes (host libm draws) are compared
BITWISE; the on-device Gaussian variant (CUDA log/cos) within 2-4 ulp."""
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.pyoracle import F32, F64, GAUSSIAN, RADEMACHER  # noqa: E402

GOLD = np.load(Path(__file__).with_name("golden") / "reference_golden.npz")


@pytest.fixture(scope="module")
def sd():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2505_11564_b200 as sd
    return sd


def ulps(a, b):
    a = np.asarray(a, np.float64).view(np.int64)
    b = np.asarray(b, np.float64).view(np.int64)
    return np.abs(a - b)


@pytest.mark.parametrize("dim", [4, 5, 129, 1025, 2050, 5000])
@pytest.mark.parametrize("workers", [1, 3])
def test_probe_parity(sd, dim, workers):
    pool = sd.make_pool(dim, workers)
    for prec in (F32, F64):
        for seed in (42, 99):
            got = sd.gather(pool, sd.draw_probe(pool, None, prec, seed=seed, distribution=sd.RADEMACHER))
            assert np.array_equal(got, GOLD[f"probe_rad_{dim}_{prec}_{seed}"])
            # Gaussian probes are bit-exact (host libm draws, rng.hpp:37-41)
            g = sd.gather(pool, sd.draw_probe(pool, None, prec, seed=seed, distribution=sd.GAUSSIAN))
            ref = GOLD[f"probe_gauss_{dim}_{prec}_{seed}"]
            assert np.array_equal(g, ref)
            # the on-device variant (CUDA log/cos) stays within a few ulp
            g = sd.gather(pool, sd.draw_probe(pool, None, prec, seed=seed, distribution=sd.GAUSSIAN_DEVICE))
            if prec == F32:
                assert np.max(np.abs(g - ref) / np.abs(ref)) <= 2 * 2.0 ** -24
            else:
                assert ulps(g, ref).max() <= 4
    v = sd.gather(sd.make_pool(5, 2), sd.draw_probe(sd.make_pool(5, 2), None, F64, distribution=sd.ONE_HOT,
                                                     one_hot_index=2, normalize=False))
    assert np.array_equal(v, GOLD["probe_onehot_5_2"])
    with pytest.raises(sd.ArgumentError):
        sd.draw_probe(sd.make_pool(5, 2), None, F64, distribution=sd.ONE_HOT, one_hot_index=5)


@pytest.mark.parametrize("dim", [1000, 1025, 5000, 70001])
def test_dot_axpy_scale_bitwise(sd, oracle, dim):
    for prec in (F32, F64):
        a = oracle.gaussian_fill(21, 0, dim)
        b = oracle.gaussian_fill(22, 0, dim)
        if prec == F32:
            a = a.astype(np.float32).astype(np.float64)
            b = b.astype(np.float32).astype(np.float64)
        ref_dot = GOLD[f"dot_{dim}_{prec}"][0]
        for workers in (1, 2, 3, 7):
            pool = sd.make_pool(dim, workers)
            A, B = sd.scatter(pool, a, prec), sd.scatter(pool, b, prec)
            d = sd.dot(pool, A, B)
            assert np.float64(d).view(np.int64) == np.float64(ref_dot).view(np.int64), (workers, prec)
            assert sd.dot(pool, B, A) == d
            assert np.array_equal(sd.gather(pool, sd.axpy(pool, 0.7, A, B)), GOLD[f"axpy_{dim}_{prec}"])
            assert np.array_equal(sd.gather(pool, sd.scale(pool, A, -1.25)), GOLD[f"scale_{dim}_{prec}"])


def test_vector_errors(sd):
    p3, p4 = sd.make_pool(3, 1), sd.make_pool(4, 1)
    a = sd.scatter(p3, [1, 2, 3], F64)
    b = sd.scatter(p4, [1, 2, 3, 4], F64)
    with pytest.raises(sd.LayoutError):
        sd.dot(p3, a, b)
    with pytest.raises(sd.LayoutError):
        sd.dot(p3, a, sd.scatter(p3, [1, 2, 3], F32))
    with pytest.raises(sd.ArgumentError):
        sd.scale(p3, a, float("nan"))
    assert sd.dot(p3, a, sd.scatter(p3, [4, 5, 6], F64)) == 32.0
    assert sd.norm2(sd.make_pool(2, 2), sd.scatter(sd.make_pool(2, 2), [3, 4], F64)) == 5.0


def test_dense_apply_bitwise(sd, oracle):
    W = sd.wigner_dense(512, 1.0, 0)
    assert np.array_equal(W, oracle.wigner(512, 1.0, 0))
    op = sd.dense_operator(W)
    for prec in (F32, F64):
        x = oracle.draw_probe(512, 7, GAUSSIAN, prec=prec)
        for workers in (1, 5):
            pool = sd.make_pool(512, workers)
            y = sd.gather(pool, op.apply(pool, sd.scatter(pool, x, prec)))
            assert np.array_equal(y, GOLD[f"wigner512_apply_{prec}"])
    with pytest.raises(sd.LayoutError):
        op.apply(sd.make_pool(5, 1), sd.scatter(sd.make_pool(5, 1), np.ones(5), F64))


@pytest.mark.parametrize("prec", [F32, F64])
@pytest.mark.parametrize("reorth", [0, 1])
def test_lanczos_dense_bitwise(sd, prec, reorth):
    S = sd.spiked_dense(256, 1.0, [50.0, -50.0], 5)
    op = sd.dense_operator(S)
    cfg = sd.LanczosConfig(k_max=25, reorthogonalize=reorth, prec=prec,
                           probe=sd.ProbeSpec(seed=42, distribution=RADEMACHER))
    r = sd.lanczos_run(op, cfg)
    assert np.array_equal(r.alphas, GOLD[f"lanczos_spiked256_{prec}_{reorth}_1_alpha"])
    assert np.array_equal(r.betas, GOLD[f"lanczos_spiked256_{prec}_{reorth}_1_beta"])
    # Gaussian probe (the reference's default distribution): bit-exact too
    cfg.probe = sd.ProbeSpec(seed=42, distribution=GAUSSIAN)
    r = sd.lanczos_run(op, cfg)
    assert np.array_equal(r.alphas, GOLD[f"lanczos_spiked256_{prec}_{reorth}_0_alpha"])
    assert np.array_equal(r.betas, GOLD[f"lanczos_spiked256_{prec}_{reorth}_0_beta"])


@pytest.mark.parametrize("P", [3 * 1024 * 1024 + 77, 1000003])
@pytest.mark.parametrize("reorth", [0, 1])
def test_lanczos_large_diag_bitwise(sd, oracle, P, reorth):
    """Engine at multi-million P (many grid blocks, ragged last block) on a
    diagonal operator, bitwise against the oracle recurrence."""
    d64 = np.linspace(-3.0, 5.0, P).astype(np.float32).astype(np.float64)
    d = torch.tensor(d64, dtype=torch.float32, device="cuda")

    k = 12
    cfg = sd.LanczosConfig(k_max=k, reorthogonalize=reorth, prec=F32,
                           probe=sd.ProbeSpec(seed=7, distribution=RADEMACHER))
    op = sd.diag_operator(d)
    r = sd.lanczos_run(op, cfg)
    ref = oracle.lanczos_diag(d64, k, reorth=bool(reorth), seed=7)
    assert np.array_equal(r.alphas, ref["alphas"])
    assert np.array_equal(r.betas, ref["betas"])


def test_ritz_matches_oracle(sd, oracle):
    S = oracle.spiked(128, 1.0, [40.0, -35.0], 2)
    r = oracle.lanczos_dense(S, 40, reorth=True)
    mine = sd.ritz_decompose(r["alphas"], r["betas"])
    v, w = oracle.ritz(r["alphas"], r["betas"])
    assert np.max(np.abs(mine.values - v)) <= 1e-12 * np.max(np.abs(v))
    assert np.max(np.abs(mine.weights - w)) <= 1e-12
    assert mine.residual <= 1e-12 and abs(mine.weights.sum() - 1) <= 1e-12


def test_f32_rounding_edge_cases(sd):
    # the reduced-precision axpy rounds f64 -> f32 on the integer pipe in the
    # fp32 normal range; it must equal IEEE round-to-nearest-even everywhere
    # (ties, carries into the exponent, overflow, subnormal and zero results)
    import ctypes as C
    rng = np.random.default_rng(7)
    n = 1 << 20
    e = rng.integers(-150, 128, n)
    y = (rng.standard_normal(n) * np.exp2(e.astype(np.float64))).astype(np.float32)
    x = (rng.standard_normal(n) * np.exp2(rng.integers(-40, 40, n).astype(np.float64))).astype(np.float32)
    special = np.array([1.0, 1.0, -1.0, 3.4028235e38, 1.1754944e-38, 1e-45, 0.0, -0.0, 1.0, np.inf, -np.inf],
                       np.float32)
    xs = np.array([2.0 ** -24, 3 * 2.0 ** -24, -(2.0 ** -24), 1e32, -1e-45, 1e-45, 0.0, 0.0, -1.0, 1.0, 1.0],
                  np.float32)
    y[: special.size] = special
    x[: xs.size] = xs
    x[-4:] = np.float32(1e30)
    y[-4:] = np.float32(3.0e38)
    for alpha in (1.0, 0.3, -1.7e-5, 3.0e8):
        want = (y.astype(np.float64) + np.float64(alpha) * x.astype(np.float64)).astype(np.float32)
        ty, tx = torch.from_numpy(y.copy()).cuda(), torch.from_numpy(x).cuda()
        ta = torch.tensor([alpha], dtype=torch.float64, device="cuda")
        rc = sd._lib.lib().sd_k_axpy(C.c_void_p(tx.data_ptr()), C.c_void_p(ty.data_ptr()), n,
                                     C.c_void_p(ta.data_ptr()), C.c_double(1.0), sd.F32,
                                     C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
        got = ty.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), alpha


@pytest.mark.parametrize("prec", [F32, F64])
@pytest.mark.parametrize("window", [2, 5, 40])
def test_lanczos_selective_bitwise(sd, oracle, prec, window):
    # selective reorth (2x CGS over the most recent W columns, ring order) ==
    # the oracle's restatement bit for bit; orthogonality between none and full
    S = sd.spiked_dense(256, 1.0, [50.0, -50.0], 5)
    op = sd.dense_operator(S)
    cfg = sd.LanczosConfig(k_max=30, reorthogonalize=sd.REORTH_SELECTIVE, prec=prec, selective_window=window,
                           probe=sd.ProbeSpec(seed=42, distribution=RADEMACHER))
    r = sd.lanczos_run(op, cfg)
    o = oracle.lanczos_dense(S, 30, reorth=2, seed=42, dist=RADEMACHER, prec=prec, window=window)
    assert np.array_equal(r.alphas, o["alphas"]) and np.array_equal(r.betas, o["betas"])
    with pytest.raises(sd.ConfigError):
        sd.lanczos_run(op, sd.LanczosConfig(k_max=5, reorthogonalize=sd.REORTH_SELECTIVE, selective_window=1))


def test_lanczos_edge_cases(sd):
    # SPEC.md:263 identity -> alpha0 = 1, beta0 below eps, stops at k = 1 (benign breakdown)
    op = sd.dense_operator(np.eye(64))
    for prec in (F32, F64):
        r = sd.lanczos_run(op, sd.LanczosConfig(k_max=10, reorthogonalize=sd.REORTH_FULL, prec=prec,
                                                probe=sd.ProbeSpec(seed=1, distribution=RADEMACHER)))
        assert r.alphas.tolist() == [1.0] and r.betas.size == 0 and r.breakdown
    # k_max = 1: one alpha, no betas
    S = sd.spiked_dense(128, 1.0, [10.0], 2)
    r = sd.lanczos_run(sd.dense_operator(S), sd.LanczosConfig(k_max=1, prec=F64))
    assert r.alphas.size == 1 and r.betas.size == 0 and not r.breakdown
    # diag(1,2,3), q0 = (1,1,1)/sqrt(3), full ortho -> eig(T) = {1,2,3}
    op3 = sd.dense_operator(np.diag([1.0, 2.0, 3.0]))
    r = sd.lanczos_run(op3, sd.LanczosConfig(k_max=3, reorthogonalize=sd.REORTH_FULL, prec=F64,
                                             probe=sd.ProbeSpec(seed=0, distribution=RADEMACHER)))
    ritz = sd.ritz_decompose(r.alphas, r.betas)
    assert np.max(np.abs(ritz.values - [1, 2, 3])) < 1e-10 and abs(ritz.weights.sum() - 1) < 1e-12
    # a non-finite operator output -> NumericalError carrying the partial tridiagonal
    import ctypes as C

    def nan_apply(x, y, s):
        t = torch.full((64,), float("nan"), dtype=torch.float64, device="cuda")
        sd._lib.lib().sd_k_scale(C.c_void_p(t.data_ptr()), C.c_void_p(y), 64,
                                 C.c_void_p(torch.ones(1, dtype=torch.float64, device="cuda").data_ptr()), 0, F64,
                                 C.c_void_p(s))
        torch.cuda.synchronize()
        return 0
    bad = sd.custom_operator(64, nan_apply, "nan")
    with pytest.raises(sd.NumericalError) as ei:
        sd.lanczos_run(bad, sd.LanczosConfig(k_max=5, prec=F64))
    assert ei.value.result.alphas.size == 0 and ei.value.result.numerical_failure
    # dimension mismatch between operator and vector -> layout error (operators.cpp:12-17)
    pool = sd.make_pool(32, 1)
    with pytest.raises(sd.LayoutError):
        op.apply(pool, sd.draw_probe(pool, None, F64))


_WIDE_REORTH = r"""
import sys, json
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2505_11564_b200 as sd
P, k, prec = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
dt = torch.float32 if prec == 0 else torch.float64
d64 = np.linspace(-3.0, 5.0, P)
if prec == 0:
    d64 = d64.astype(np.float32).astype(np.float64)
d = torch.tensor(d64, dtype=dt, device="cuda")
cfg = sd.LanczosConfig(k_max=k, reorthogonalize=sd.REORTH_FULL, prec=prec,
                       probe=sd.ProbeSpec(seed=7, distribution=sd.RADEMACHER))
r = sd.lanczos_run(sd.diag_operator(d), cfg)
print(json.dumps({"a": [x.hex() for x in r.alphas.tolist()], "b": [x.hex() for x in r.betas.tolist()]}))
"""


@pytest.mark.parametrize("prec,k,variants", [
    (F32, 64, ("default", "0", "1000")),
    (F64, 48, ("default",)),
])
def test_lanczos_wide_reorth_bitwise(sd, oracle, prec, k, variants):
    """Full reorthogonalisation at j >= 40 stored columns over full 1024-blocks
    (P = 2^21 + 77: 2048 full grid blocks and a ragged tail) -- the path the
    bench times (k_cgs_update + k_cgs_block<T,false> beyond
    SD_CGS_FUSED_UPDATE_MAX columns, the fused in-CTA update below it) --
    bitwise against the oracle's recurrence (reduction.hpp:76-107,
    SPEC.md:260,284). SD_CGS_FUSED_UPDATE_MAX=0 forces the split kernels at
    every width, =1000 the fused kernel at every width."""
    import json
    import os
    import subprocess
    import sys
    root = str(Path(__file__).resolve().parents[1])
    P = 2 ** 21 + 77
    d64 = np.linspace(-3.0, 5.0, P)
    if prec == F32:
        d64 = d64.astype(np.float32).astype(np.float64)
    ref = oracle.lanczos_diag(d64, k, reorth=True, seed=7, prec=prec)
    assert len(ref["alphas"]) == k
    for var in variants:
        env = dict(os.environ)
        if var != "default":
            env["SD_CGS_FUSED_UPDATE_MAX"] = var
        r = subprocess.run([sys.executable, "-c", _WIDE_REORTH, root, str(P), str(k), str(prec)], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        got = json.loads(r.stdout.strip().splitlines()[-1])
        a = np.array([float.fromhex(x) for x in got["a"]])
        b = np.array([float.fromhex(x) for x in got["b"]])
        assert np.array_equal(a, ref["alphas"]), (var, np.max(np.abs(a - ref["alphas"])))
        assert np.array_equal(b, ref["betas"]), (var, np.max(np.abs(b - ref["betas"])))


@pytest.mark.parametrize("prec", [F32, F64])
def test_gaussian_probe_bitwise_large(sd, oracle, prec):
    """SD_GAUSSIAN (the reference's default probe, sharded.hpp:36-38) at 9M
    elements over 3 ragged workers -- several pinned staging chunks per shard
    -- equals the oracle's glibc draws bit for bit (rng.hpp:37-41, round_elem)."""
    P = 9_000_011
    pool = sd.make_pool(P, 3)
    got = sd.gather(pool, sd.draw_probe(pool, None, prec, seed=2718, distribution=sd.GAUSSIAN, normalize=False))
    ref = oracle.gaussian_fill(2718, 0, P)
    if prec == F32:
        ref = ref.astype(np.float32).astype(np.float64)
    assert np.array_equal(got, ref)
