"""GPU MLP HVP engine (SPEC.md:179 mlp(layer_widths), tanh + mse) vs the f64
oracle restatement (oracle/src/models.cpp build_mlp), finite differences of
the oracle's gradients (acceptance 1), symmetry, linearity and
the batch-size weighting of batched_hvp."""
import numpy as np
import pytest

from oracle.pyoracle import F32

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2505_11564_b200 import mlp
    return mlp


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def setup(widths, n, seed):
    rng = np.random.default_rng(seed)
    from paper_2505_11564_b200 import mlp
    P = mlp.param_count(widths)
    th = f32(rng.standard_normal(P) * 0.5)
    X = f32(rng.standard_normal((n, widths[0])))
    Y = f32(rng.standard_normal((n, widths[-1])))
    return rng, P, th, X, Y


@pytest.mark.parametrize("widths,n", [([4, 8, 1], 10), ([16, 32, 32, 4], 64), ([5, 7, 3], 33), ([64, 256, 128, 10], 200)])
def test_mlp_hvp_matches_oracle(M, oracle, widths, n):
    rng, P, th, X, Y = setup(widths, n, len(widths) * 7 + n)
    assert P == oracle.mlp_param_count(widths)
    eng = M.MlpHvp(widths, torch.tensor(th, dtype=torch.float32, device="cuda"), n_max=n, x=X, y=Y)
    for _ in range(3):
        v = f32(rng.standard_normal(P))
        got = eng.hvp(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()
        want = oracle.mlp_hvp(widths, th, X, Y, v)
        # bar: 1e-5, or -- where the model amplifies rounding (wide tanh layers,
        # many samples) -- 32x the oracle's own f32-per-node error: a 3xTF32
        # product carries ~2^-21 relative error (tf32 residual of the residual
        # and the dropped lo*lo term) against 2^-24 for an exactly rounded one
        f32_err = np.linalg.norm(oracle.mlp_hvp(widths, th, X, Y, v, prec=F32) - want) / np.linalg.norm(want)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < max(1e-5, 32 * f32_err)
    assert eng.loss() > 0


def test_mlp_finite_differences_and_symmetry(M, oracle):
    # acceptance 1: MLP [4,8,1] Hv vs central differences (eps 1e-4, f64 gradients)
    widths = [4, 8, 1]
    rng, P, th, X, Y = setup(widths, 10, 3)
    eng = M.MlpHvp(widths, torch.tensor(th, dtype=torch.float32, device="cuda"), n_max=16, x=X, y=Y)
    for _ in range(20):
        v = f32(rng.standard_normal(P))
        hv = eng.hvp(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()
        fd = (oracle.mlp_grad(widths, th + 1e-4 * v, X, Y) - oracle.mlp_grad(widths, th - 1e-4 * v, X, Y)) / 2e-4
        assert np.linalg.norm(hv - fd) / np.linalg.norm(fd) < 1e-5
    u, w = f32(rng.standard_normal(P)), f32(rng.standard_normal(P))
    hu = eng.hvp(torch.tensor(u, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    hw = eng.hvp(torch.tensor(w, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    assert abs(hu @ w - u @ hw) < 1e-5 * np.linalg.norm(hu) * np.linalg.norm(w)
    lin = eng.hvp(torch.tensor(0.5 * u - 2.0 * w, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    assert np.linalg.norm(lin - (0.5 * hu - 2.0 * hw)) < 1e-5 * np.linalg.norm(lin)


def test_mlp_batched_hvp_weighting(M):
    # batches of sizes 1 and 3 == the concatenated 4-sample batch
    widths = [6, 12, 2]
    rng, P, th, X, Y = setup(widths, 4, 11)
    theta = torch.tensor(th, dtype=torch.float32, device="cuda")
    eng = M.MlpHvp(widths, theta, n_max=4)
    v = torch.tensor(f32(rng.standard_normal(P)), dtype=torch.float32, device="cuda")
    split = M.batched_hvp(eng, [(X[:1], Y[:1]), (X[1:], Y[1:])], v).double().cpu().numpy()
    whole = M.batched_hvp(eng, [(X, Y)], v).double().cpu().numpy()
    assert np.linalg.norm(split - whole) / np.linalg.norm(whole) < 1e-5


def test_mlp_lanczos_spectrum(M, oracle):
    # the MLP operator through the device Lanczos engine: full-reorth Ritz values
    # of a tiny model match the eigenvalues of the oracle's dense f64 Hessian
    import paper_2505_11564_b200 as sd
    widths = [3, 5, 2]
    rng, P, th, X, Y = setup(widths, 12, 5)
    eng = M.MlpHvp(widths, torch.tensor(th, dtype=torch.float32, device="cuda"), n_max=12, x=X, y=Y)
    H = np.stack([oracle.mlp_hvp(widths, th, X, Y, np.eye(P)[i]) for i in range(P)])
    lam = np.linalg.eigvalsh(0.5 * (H + H.T))
    cfg = sd.LanczosConfig(k_max=P, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                           probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
    res = sd.lanczos_run(eng.operator(), cfg)
    spec = sd.ritz_decompose(res.alphas, res.betas)
    scale = np.abs(lam).max()
    for t in spec.values:
        assert np.min(np.abs(lam - t)) < 1e-4 * scale
