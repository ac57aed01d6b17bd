"""Tree-mode Lanczos (SD_REDUCE_TREE: fused TMA-staged GEMV passes with
fixed-order warp-shuffle + block reductions, sd_lanczos_tree.cu) against the
ordered mode (the reference's 1024-block fold, itself bitwise against the
oracle): the same recurrence up to rounding.

Tolerances: f64 storage -- alpha/beta within 1e-12 of ordered mode relative to
||T||; f32 storage -- within 2e-6 (every stored element is rounded to f32, and
the two modes round different intermediate vectors). Without full
reorthogonalisation (none / selective) the recurrence itself amplifies
rounding differences once Ritz values converge (ghosts), so those runs are
compared over their first 10 steps. Tree mode is deterministic: reruns are
bitwise identical.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sd():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2505_11564_b200 as sd
    return sd


def tdiff(a, b, steps=None):
    assert a.alphas.size == b.alphas.size and a.betas.size == b.betas.size
    aa, ab = a.alphas[:steps], a.betas[:steps]
    ba, bb = b.alphas[:steps], b.betas[:steps]
    na = max(np.max(np.abs(ba)), np.max(np.abs(bb)) if bb.size else 0.0)
    da = np.max(np.abs(aa - ba))
    db = np.max(np.abs(ab - bb)) if bb.size else 0.0
    return max(da, db) / na


@pytest.mark.parametrize("prec,tol", [(1, 1e-12), (0, 2e-6)])
@pytest.mark.parametrize("reorth,window", [(0, 0), (1, 0), (2, 5)])
def test_tree_matches_ordered_dense(sd, prec, tol, reorth, window):
    S = sd.spiked_dense(256, 1.0, [50.0, -50.0], 5)
    op = sd.dense_operator(S)
    base = dict(k_max=25, reorthogonalize=reorth, prec=prec, selective_window=window,
                probe=sd.ProbeSpec(seed=42, distribution=sd.RADEMACHER))
    a = sd.lanczos_run(op, sd.LanczosConfig(**base))
    b = sd.lanczos_run(op, sd.LanczosConfig(**base, reduction=sd.REDUCE_TREE))
    steps = None if reorth == 1 else 10
    assert tdiff(b, a, steps) <= tol, tdiff(b, a, steps)
    c = sd.lanczos_run(op, sd.LanczosConfig(**base, reduction=sd.REDUCE_TREE))
    assert np.array_equal(b.alphas, c.alphas) and np.array_equal(b.betas, c.betas)  # deterministic


@pytest.mark.parametrize("prec,tol,k", [(1, 1e-12, 40), (0, 2e-6, 110)])
def test_tree_matches_ordered_large_diag(sd, prec, tol, k):
    # many tiles per CTA, a ragged last tile, > 128 columns (2-stage ring) in f32
    P = 2 ** 21 + 77
    dt = torch.float32 if prec == 0 else torch.float64
    d = torch.linspace(-3.0, 5.0, P, dtype=torch.float64, device="cuda").to(dt)
    op = sd.diag_operator(d)
    base = dict(k_max=k, reorthogonalize=sd.REORTH_FULL, prec=prec,
                probe=sd.ProbeSpec(seed=7, distribution=sd.RADEMACHER))
    a = sd.lanczos_run(op, sd.LanczosConfig(**base))
    b = sd.lanczos_run(op, sd.LanczosConfig(**base, reduction=sd.REDUCE_TREE))
    assert tdiff(b, a) <= tol, tdiff(b, a)
    # the Ritz values (what SLQ consumes) agree as closely
    ra, rb = sd.ritz_decompose(a.alphas, a.betas), sd.ritz_decompose(b.alphas, b.betas)
    assert np.max(np.abs(ra.values - rb.values)) <= tol * 8.0


def test_tree_basis_is_orthonormal(sd):
    # full reorth in tree mode keeps the basis orthonormal to f32 working precision
    P = 300001
    d = torch.linspace(-1.0, 1.0, P, device="cuda")
    cfg = sd.LanczosConfig(k_max=60, reorthogonalize=sd.REORTH_FULL, prec=sd.F32, reduction=sd.REDUCE_TREE,
                           probe=sd.ProbeSpec(seed=3, distribution=sd.RADEMACHER))
    r = sd.lanczos_run(sd.diag_operator(d), cfg, with_basis=True)
    Q = r.basis
    G = Q @ Q.T
    assert np.max(np.abs(G - np.eye(G.shape[0]))) < 1e-5


def test_tree_workers_match_one_worker(sd):
    # sharded tree mode: per-rank fixed-order sums, all-gathered and folded in
    # rank order; 4 ragged in-process workers vs one
    S = sd.spiked_dense(300, 1.0, [40.0, -40.0], 3)
    op = sd.dense_operator(S)
    cfg = sd.LanczosConfig(k_max=14, reorthogonalize=sd.REORTH_FULL, prec=sd.F64, reduction=sd.REDUCE_TREE,
                           probe=sd.ProbeSpec(seed=42, distribution=sd.RADEMACHER))
    one = sd.lanczos_run(op, cfg)
    lay = sd.split_evenly(300, 4)
    out = sd.run_workers(4, lambda r, c: sd.lanczos_run(op, cfg, layout=lay, comm=c))
    for r in out:
        assert np.array_equal(r.alphas, out[0].alphas)
        assert tdiff(r, one) <= 1e-12


def test_tree_c1_slq_vs_cpu_oracle(sd, oracle):
    # BASELINE configs[0] in tree mode: same tolerances as the ordered-mode check
    from paper_2505_11564_b200 import gpt
    import slq_c1
    cpu = slq_c1.cpu_run(oracle)
    eng = gpt.GptHvp(slq_c1.C1, slq_c1.B, slq_c1.S, init_seed=0)
    cfg = sd.LanczosConfig(k_max=slq_c1.K, reorthogonalize=sd.REORTH_FULL, prec=sd.F32, reduction=sd.REDUCE_TREE,
                           probe=sd.ProbeSpec(seed=slq_c1.SEED, distribution=sd.RADEMACHER))
    res = sd.lanczos_run(eng.operator(), cfg)
    rz = sd.ritz_decompose(res.alphas, res.betas)
    err = slq_c1.compare((res.alphas, res.betas, rz.values, rz.weights), cpu)
    print("C1 tree mode:", err)


def test_tree_rejects_too_many_columns(sd):
    op = sd.dense_operator(np.eye(512))
    with pytest.raises(sd.ConfigError):
        sd.lanczos_run(op, sd.LanczosConfig(k_max=300, reorthogonalize=sd.REORTH_FULL, reduction=sd.REDUCE_TREE))


def test_tree_on_the_bench_operator(sd):
    """The bench path itself: GPT-2-small (124M parameters, one 1024-token
    sequence) HVP driving full-reorth Lanczos in tree mode vs ordered mode --
    the same Hv (deterministic engine), only the reductions differ: alpha/beta
    within 2e-6 of ||T|| over 10 steps, basis orthonormal."""
    from paper_2505_11564_b200 import gpt
    eng = gpt.GptHvp(gpt.GPT2_SMALL, 1, 1024, init_seed=0)
    base = dict(k_max=10, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
    a = sd.lanczos_run(eng.operator(), sd.LanczosConfig(**base))
    b = sd.lanczos_run(eng.operator(), sd.LanczosConfig(**base, reduction=sd.REDUCE_TREE))
    assert tdiff(b, a) <= 2e-6, tdiff(b, a)
    L = sd.Lanczos(eng.operator(), sd.LanczosConfig(**base, reduction=sd.REDUCE_TREE))
    while not L.step():
        pass
    assert L.loss_of_orthogonality() < 1e-5
    L.close()
    eng.close()


def test_tree_edge_cases(sd):
    # SPEC.md:263 identity: alpha0 = 1, beta0 below eps -> benign breakdown at k = 1;
    # diag(1,2,3) recovers its eigenvalues; a short vector (P < one 128-element tile)
    for prec in (sd.F32, sd.F64):
        r = sd.lanczos_run(sd.dense_operator(np.eye(64)),
                           sd.LanczosConfig(k_max=10, reorthogonalize=sd.REORTH_FULL, prec=prec,
                                            reduction=sd.REDUCE_TREE,
                                            probe=sd.ProbeSpec(seed=1, distribution=sd.RADEMACHER)))
        assert r.alphas.size == 1 and abs(r.alphas[0] - 1.0) < 1e-6 and r.breakdown
    r = sd.lanczos_run(sd.dense_operator(np.diag([1.0, 2.0, 3.0])),
                       sd.LanczosConfig(k_max=3, reorthogonalize=sd.REORTH_FULL, prec=sd.F64, reduction=sd.REDUCE_TREE,
                                        probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER)))
    ritz = sd.ritz_decompose(r.alphas, r.betas)
    assert np.max(np.abs(ritz.values - [1, 2, 3])) < 1e-10
    # a non-finite operator output -> NumericalError with the partial tridiagonal
    import ctypes as C

    def nan_apply(x, y, s):
        t = torch.full((64,), float("nan"), dtype=torch.float64, device="cuda")
        sd._lib.lib().sd_k_scale(C.c_void_p(t.data_ptr()), C.c_void_p(y), 64,
                                 C.c_void_p(torch.ones(1, dtype=torch.float64, device="cuda").data_ptr()), 0, sd.F64,
                                 C.c_void_p(s))
        torch.cuda.synchronize()
        return 0
    with pytest.raises(sd.NumericalError):
        sd.lanczos_run(sd.custom_operator(64, nan_apply, "nan"),
                       sd.LanczosConfig(k_max=5, prec=sd.F64, reduction=sd.REDUCE_TREE))
