"""Pins the CPU oracle (oracle/src) before anything is checked against it:
Appendix-A golden values of the compiled reference, the committed reference
fixtures (tests/golden/reference_golden.npz), the reference's own 45 doctest
cases, SPEC known answers, and finite differences for the HVP."""
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle.pyoracle import F32, F64, GAUSSIAN, ONE_HOT, RADEMACHER, OracleError

GOLD = np.load(Path(__file__).with_name("golden") / "reference_golden.npz")


def hx(x):
    return hex(struct.unpack("<Q", struct.pack("<d", x))[0])


def test_appendix_a_golden(oracle):
    # SURVEY.md Appendix A, captured from the compiled reference
    assert oracle.keyed_counter(42, 0) == 0x57E1FABA65107204
    assert oracle.mix64(0) == 0xE220A8397B1DCDAF
    assert [hx(oracle.gaussian(42, i)) for i in range(4)] == [
        "0xbfe03f92665aa395", "0x3fdc38ee63857bdb", "0x3f95fc5b483df6d6", "0x3fd08e56d93852e4"]
    assert "".join("+" if oracle.rademacher(7, i) > 0 else "-" for i in range(16)) == "+-++-++-+++--+--"
    assert [hx(x) for x in oracle.draw_probe(4, 42)] == [
        "0xbfe68a2d7577e812", "0x3fe3933aac6a566a", "0x3f9e7faebd8f7d95", "0x3fd6f771ad2d6a22"]
    assert [hx(x) for x in oracle.draw_probe(4, 42, prec=F32)] == [
        "0xbfe68a2d80000000", "0x3fe3933aa0000000", "0x3f9e7faec0000000", "0x3fd6f771c0000000"]


@pytest.mark.parametrize("dim", [4, 5, 129, 1025, 2050, 5000])
def test_probes_match_reference_fixtures(oracle, dim):
    for prec in (F32, F64):
        for dist, name in ((GAUSSIAN, "gauss"), (RADEMACHER, "rad")):
            for seed in (42, 99):
                got = oracle.draw_probe(dim, seed, dist, prec=prec)
                assert np.array_equal(got, GOLD[f"probe_{name}_{dim}_{prec}_{seed}"])
    assert np.array_equal(oracle.draw_probe(5, 0, ONE_HOT, 2, normalize=False), GOLD["probe_onehot_5_2"])


@pytest.mark.parametrize("dim", [1000, 1025, 5000, 70001])
def test_vector_ops_match_reference_fixtures(oracle, dim):
    for prec in (F32, F64):
        a = oracle.gaussian_fill(21, 0, dim)
        b = oracle.gaussian_fill(22, 0, dim)
        if prec == F32:
            a = a.astype(np.float32).astype(np.float64)
            b = b.astype(np.float32).astype(np.float64)
        d = oracle.dot(a, b)
        assert hx(d) == hx(GOLD[f"dot_{dim}_{prec}"][0])
        assert np.array_equal(oracle.axpy(0.7, a, b, prec), GOLD[f"axpy_{dim}_{prec}"])
        assert np.array_equal(oracle.scale(a, -1.25, prec), GOLD[f"scale_{dim}_{prec}"])


def test_dense_and_lanczos_match_reference_fixtures(oracle):
    assert np.array_equal(oracle.wigner(64, 1.0, 3), GOLD["wigner_64_1_3"])
    assert np.array_equal(oracle.spiked(128, 1.0, [40.0, -35.0], 2), GOLD["spiked_128_1_2"])
    W = oracle.wigner(512, 1.0, 0)
    for prec in (F32, F64):
        x = oracle.draw_probe(512, 7, GAUSSIAN, prec=prec)
        assert np.array_equal(oracle.dense_apply(W, x, prec), GOLD[f"wigner512_apply_{prec}"])
    S = oracle.spiked(256, 1.0, [50.0, -50.0], 5)
    for prec in (F32, F64):
        for reorth in (0, 1):
            for dist in (0, 1):
                res = oracle.lanczos_dense(S, 25, reorth=bool(reorth), seed=42, dist=dist, prec=prec)
                assert np.array_equal(res["alphas"], GOLD[f"lanczos_spiked256_{prec}_{reorth}_{dist}_alpha"])
                assert np.array_equal(res["betas"], GOLD[f"lanczos_spiked256_{prec}_{reorth}_{dist}_beta"])


def test_reference_doctest_binaries(reference):
    # the reference's own 45 test cases, built against oracle/shims
    ref = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
    total = 0
    for t in ("test_sharded_core", "test_runtime", "test_operators"):
        r = subprocess.run([str(ref / t)], capture_output=True, text=True, cwd=ref, timeout=300)
        assert r.returncode == 0, r.stdout[-2000:]
        total += int(r.stdout.split("test cases: ")[1].split()[0])
    assert total == 45


def test_oracle_equals_live_reference(oracle, reference):
    for dim, workers in ((1234, 4), (4097, 5), (2050, 8)):
        for prec in (F32, F64):
            a = reference.draw_probe(dim, workers, 61, GAUSSIAN, prec=prec)
            b = reference.draw_probe(dim, workers, 62, RADEMACHER, prec=prec)
            assert np.array_equal(a, oracle.draw_probe(dim, 61, GAUSSIAN, prec=prec))
            assert hx(reference.dot(a, b, workers, prec)) == hx(oracle.dot(a, b))
            assert np.array_equal(reference.axpy(2.5, a, b, workers, prec), oracle.axpy(2.5, a, b, prec))


def test_layout_and_partials(oracle):
    for dim in (1, 2, 7, 10, 1000):
        for n in (1, 2, 3, 4, 8, 16):
            rs = oracle.split_evenly(dim, n)
            assert len(rs) == min(dim, n)
            sizes = [e - b for b, e in rs]
            assert sum(sizes) == dim and max(sizes) - min(sizes) <= 1
    with pytest.raises(OracleError) as ei:
        oracle.validate_layout(10, [(0, 4), (5, 10)])
    assert ei.value.kind == "layout_error"
    # blocked partials reproduce the fixed DAG for any split (reduction.hpp:76-107)
    P = 5000
    a = oracle.gaussian_fill(3, 0, P)
    b = oracle.gaussian_fill(4, 0, P)
    ref = oracle.dot(a, b)
    for n in (1, 2, 3, 7, 8):
        rs = oracle.split_evenly(P, n)
        parts = [oracle.dot_partial(s, e, P, a[s:e], b[s:e]) for s, e in rs]
        assert hx(oracle.combine_partials(P, rs, parts)) == hx(ref)
    with pytest.raises(OracleError) as ei:
        rs = oracle.split_evenly(P, 2)
        parts = [oracle.dot_partial(s, e, P, a[s:e], b[s:e]) for s, e in rs]
        oracle.combine_partials(P, rs[::-1], parts[::-1])
    assert ei.value.kind == "protocol_error"


def test_lanczos_known_answers(oracle):
    # identity: alpha0 = 1, beta0 ~ 0, stops at k = 1
    r = oracle.lanczos_dense(np.eye(16), 10)
    assert len(r["alphas"]) == 1 and abs(r["alphas"][0] - 1) < 1e-15 and r["breakdown"]
    # diag(1,2,3) full reorth -> eig(T) = {1,2,3}
    r = oracle.lanczos_dense(np.diag([1.0, 2.0, 3.0]), 3, reorth=True)
    v, w = oracle.ritz(r["alphas"], r["betas"])
    assert np.max(np.abs(v - [1, 2, 3])) < 1e-10 and abs(w.sum() - 1) < 1e-12
    # exact recovery, P <= 64, k = P, full ortho
    A = oracle.wigner(64, 1.0, 11)
    r = oracle.lanczos_dense(A, 64, reorth=True)
    v, _ = oracle.ritz(r["alphas"], r["betas"])
    assert np.max(np.abs(v - np.linalg.eigvalsh(A))) < 1e-8
    # Gauss moment matching sum w theta^m = q0^T A^m q0, m <= 2k-1
    A = oracle.wigner(256, 1.0 / 16, 4)
    for k in (5, 10):
        r = oracle.lanczos_dense(A, k, reorth=True, basis=True)
        v, w = oracle.ritz(r["alphas"], r["betas"])
        q0 = r["basis"][0]
        x = q0.copy()
        for m in range(2 * k):
            lhs = float(np.sum(w * v ** m))
            rhs = float(q0 @ x)
            assert abs(lhs - rhs) <= 1e-8 * max(1.0, abs(rhs))
            x = A @ x
    # ghosts (PAPER Fig. 3): once the outlier Ritz value converges, the
    # no-ortho run duplicates it; full reorth never does
    A = oracle.spiked(256, 1.0, [100.0, -100.0], 5)
    no = oracle.ritz(*[oracle.lanczos_dense(A, 40, reorth=False)[k] for k in ("alphas", "betas")])[0]
    fu = oracle.ritz(*[oracle.lanczos_dense(A, 40, reorth=True)[k] for k in ("alphas", "betas")])[0]
    gap = lambda v: np.min(np.diff(v[-3:]))  # noqa: E731
    assert gap(no) < 1e-9 * (no[-1] - no[0]) < gap(fu)


def test_ritz_and_density_known_answers(oracle):
    v, w = oracle.ritz([3.5], [])
    assert v[0] == 3.5 and w[0] == 1.0
    v, w = oracle.ritz([0.0, 0.0], [1.0])
    assert np.allclose(v, [-1, 1], atol=1e-15) and np.allclose(w, [0.5, 0.5], atol=1e-15)
    g, d, s = oracle.smooth_density([0.0], [1.0], 1.0, 1001)
    assert abs(d[500] - 1 / np.sqrt(2 * np.pi)) < 1e-15 and abs(np.trapezoid(d, g) - 1) < 1e-2


def test_mlp_hvp_finite_differences(oracle):
    # MLP [4,8,1] hvp vs central differences of gradients, eps=1e-4, rel < 1e-5
    wd = [4, 8, 1]
    P = oracle.mlp_param_count(wd)
    rng = np.random.default_rng(0)
    th = rng.standard_normal(P) * 0.5
    X = rng.standard_normal((10, 4))
    Y = rng.standard_normal((10, 1))
    for t in range(5):
        v = rng.standard_normal(P)
        hv = oracle.mlp_hvp(wd, th, X, Y, v)
        fd = (oracle.mlp_grad(wd, th + 1e-4 * v, X, Y) - oracle.mlp_grad(wd, th - 1e-4 * v, X, Y)) / 2e-4
        assert np.linalg.norm(hv - fd) / np.linalg.norm(fd) < 1e-5
    # symmetry and linearity
    u, w = rng.standard_normal(P), rng.standard_normal(P)
    assert abs(oracle.mlp_hvp(wd, th, X, Y, u) @ w - u @ oracle.mlp_hvp(wd, th, X, Y, w)) < 1e-8 * np.linalg.norm(u) * np.linalg.norm(w)
    lin = oracle.mlp_hvp(wd, th, X, Y, 0.3 * u - 1.7 * w)
    assert np.linalg.norm(lin - (0.3 * oracle.mlp_hvp(wd, th, X, Y, u) - 1.7 * oracle.mlp_hvp(wd, th, X, Y, w))) < 1e-10 * np.linalg.norm(lin)


TINY = dict(n_layer=2, d=16, n_head=2, ff=64, vocab=32, ctx=8)


def test_gpt_hvp_finite_differences_and_torch(oracle):
    import torch
    import torch_gpt
    P = oracle.gpt_param_count(TINY)
    th = oracle.gpt_init(TINY, 0, 0.1, 0.1)
    tok, tgt = oracle.gpt_batch(TINY, 2, 8)
    v = oracle.draw_probe(P, 3, RADEMACHER)
    hv = oracle.gpt_hvp(TINY, th, tok, tgt, 2, 8, v)
    fd = (oracle.gpt_grad(TINY, th + 1e-4 * v, tok, tgt, 2, 8) - oracle.gpt_grad(TINY, th - 1e-4 * v, tok, tgt, 2, 8)) / 2e-4
    assert np.linalg.norm(hv - fd) / np.linalg.norm(fd) < 1e-5
    ht = torch_gpt.hvp(TINY, torch.tensor(th), torch.tensor(tok.astype(np.int64)), torch.tensor(tgt.astype(np.int64)),
                       2, 8, torch.tensor(v)).numpy()
    assert np.linalg.norm(ht - hv) / np.linalg.norm(hv) < 1e-12


@pytest.mark.parametrize("kv", [0, 2])
def test_torch_llama_restatement_matches_oracle(oracle, kv):
    # the float64 torch Llama restatement (RMSNorm, rotate-half RoPE, GQA,
    # SwiGLU, untied head) that pins the GPU engine at S >= 1024 equals the
    # oracle's Graph HVP (oracle/src/models.cpp build_llama) at small shapes
    import torch
    import torch_gpt
    cfg = dict(n_layer=2, d=64, n_head=8, ff=96, vocab=96, ctx=32, arch=1, rope_base=10000, n_kv_head=kv)
    th = oracle.gpt_init(cfg, 0, 0.1, 0.1)
    tok, tgt = oracle.gpt_batch(cfg, 2, 16)
    v = oracle.draw_probe(th.size, 3, RADEMACHER)
    hv = oracle.gpt_hvp(cfg, th, tok, tgt, 2, 16, v)
    ht = torch_gpt.llama_hvp(cfg, torch.tensor(th), torch.tensor(tok.astype(np.int64)),
                             torch.tensor(tgt.astype(np.int64)), 2, 16, torch.tensor(v)).numpy()
    assert np.linalg.norm(ht - hv) / np.linalg.norm(hv) < 1e-12


def test_gpt_batched_hvp_weighting(oracle):
    # batches of sizes 1 and 3 == one concatenated 4-sample batch, within 1e-10
    P = oracle.gpt_param_count(TINY)
    th = oracle.gpt_init(TINY, 0, 0.1, 0.1)
    tok, tgt = oracle.gpt_batch(TINY, 4, 8)
    v = oracle.draw_probe(P, 5, RADEMACHER)
    whole = oracle.gpt_hvp(TINY, th, tok, tgt, 4, 8, v)
    split = oracle.gpt_batched_hvp(TINY, th, [(1, tok[:8], tgt[:8]), (3, tok[8:], tgt[8:])], 8, v)
    assert np.linalg.norm(split - whole) / np.linalg.norm(whole) < 1e-10


def test_selective_reorth_sits_between_none_and_full(oracle):
    # the oracle's selective variant: its basis loses orthogonality more slowly
    # than no reorth and a window covering the whole run equals full reorth
    from oracle.pyoracle import F64, RADEMACHER
    S = oracle.spiked(256, 1.0 / 16, [100.0, -100.0], 7)
    def lo(reorth, window=0):
        r = oracle.lanczos_dense(S, 25, reorth=reorth, seed=1, dist=RADEMACHER, prec=F64, basis=True, window=window)
        Q = r["basis"]
        G = Q @ Q.T
        return np.max(np.abs(G - np.eye(G.shape[0]))), r
    # (a local window only helps once it covers the early, converged
    # directions: W = 4 leaves this spiked run as non-orthogonal as none)
    l_none, _ = lo(0)
    l_sel, _ = lo(2, 20)
    l_full, rf = lo(1)
    assert l_full < l_sel < 1e-9 < l_none
    _, rw = lo(2, 26)
    assert np.array_equal(rw["alphas"], rf["alphas"]) and np.array_equal(rw["betas"], rf["betas"])


def test_lanczos_over_gpt_hvp_moments(oracle):
    # the CPU leg of the C1 SLQ parity check (oracle_lanczos_gpt): Gauss
    # quadrature of its tridiagonal reproduces q0^T H^m q0 for m <= 2k-1
    # (SPEC.md:348), H applied by the oracle's own HVP in f64
    import slq_c1
    cfg, B, S, k = slq_c1.C1, 2, 16, 6
    th = oracle.gpt_init(cfg, 0, 0.0, 0.0, prec=F64)
    tok, tgt = oracle.gpt_batch(cfg, B, S)
    r = oracle.lanczos_gpt(cfg, th, tok, tgt, B, S, k, reorth=True, seed=42, dist=RADEMACHER, prec=F64, hvp_prec=F64)
    v, w = oracle.ritz(r["alphas"], r["betas"])
    q0 = oracle.draw_probe(th.size, 42, RADEMACHER, prec=F64)
    x = q0.copy()
    for m in range(2 * k):
        rhs = float(q0 @ x)
        lhs = float(np.sum(w * v ** m))
        assert abs(lhs - rhs) <= 1e-8 * float(np.sum(w * np.abs(v) ** m)), m
        x = oracle.gpt_hvp(cfg, th, tok, tgt, B, S, x, prec=F64)
