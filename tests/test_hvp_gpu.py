"""GPT HVP on B200 vs (1) the f64 C++ oracle (autodiff Graph restatement),
(2) an independent float64 torch double-backward, (3) central finite
differences, plus the SPEC's HVP properties. Tolerance (north star): rel-L2
<= 1e-5 against the f64 reference for the fp32 pipeline."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def sd():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2505_11564_b200 as sd
    return sd


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


TINY = dict(n_layer=2, d=64, n_head=4, ff=256, vocab=96, ctx=32)
C1 = dict(n_layer=1, d=64, n_head=4, ff=256, vocab=64, ctx=32)


def test_layout_and_tokens_match_oracle(sd, oracle):
    from paper_2505_11564_b200 import gpt
    for cfg in (TINY, C1, gpt.GPT2_SMALL):
        assert gpt.param_count(cfg) == oracle.gpt_param_count(cfg)
    assert gpt.param_count(gpt.GPT2_SMALL) == 124439808
    lay = gpt.param_layout(TINY)
    assert lay == oracle.gpt_layout(TINY)
    tok, tgt = gpt.synthetic_tokens(TINY["vocab"], 3, 32, 1, 5)
    otok, otgt = oracle.gpt_batch(TINY, 3, 32, 1, 5)
    assert np.array_equal(tok, otok.astype(np.int32)) and np.array_equal(tgt, otgt.astype(np.int32))


@pytest.mark.parametrize("cfg,B,S", [(TINY, 2, 32), (C1, 4, 32), (dict(TINY, n_layer=1, n_head=2, d=32, ff=128), 1, 12)])
def test_hvp_vs_oracle(sd, oracle, cfg, B, S):
    from paper_2505_11564_b200 import gpt
    eng = gpt.GptHvp(cfg, B, S, init_seed=0, gain_scale=0.1, bias_scale=0.1)
    th = eng.theta_numpy()
    # synthetic init is bit-identical to the oracle's f32-rounded init
    assert np.array_equal(th, oracle.gpt_init(cfg, 0, 0.1, 0.1, prec=0))
    tok, tgt = eng.tokens_numpy()
    for seed in (3, 4):
        v = oracle.draw_probe(eng.P, seed, 1, prec=0)
        hv = eng.hvp_numpy(v)
        ref = oracle.gpt_hvp(cfg, th, tok, tgt, B, S, v)
        assert rel(hv, ref) < TOL, rel(hv, ref)
    loss = eng.loss()
    assert abs(loss - oracle.gpt_loss(cfg, th, tok, tgt, B, S)) < 1e-5


def test_hvp_finite_differences_and_properties(sd, oracle):
    from paper_2505_11564_b200 import gpt
    cfg, B, S = TINY, 2, 32
    eng = gpt.GptHvp(cfg, B, S, init_seed=1, gain_scale=0.1, bias_scale=0.1)
    th = eng.theta_numpy()
    tok, tgt = eng.tokens_numpy()
    rng = np.random.default_rng(0)
    v = rng.standard_normal(eng.P).astype(np.float32).astype(np.float64)
    hv = eng.hvp_numpy(v)
    e = 1e-4
    fd = (oracle.gpt_grad(cfg, th + e * v, tok, tgt, B, S) - oracle.gpt_grad(cfg, th - e * v, tok, tgt, B, S)) / (2 * e)
    assert rel(hv, fd) < 2e-5
    # symmetry <Hu, w> = <u, Hw> and linearity
    u = rng.standard_normal(eng.P).astype(np.float32).astype(np.float64)
    w = rng.standard_normal(eng.P).astype(np.float32).astype(np.float64)
    hu, hw = eng.hvp_numpy(u), eng.hvp_numpy(w)
    assert abs(hu @ w - u @ hw) <= 1e-5 * np.linalg.norm(hu) * np.linalg.norm(w)
    lin = eng.hvp_numpy((0.5 * u - 2.0 * w).astype(np.float32))
    assert rel(lin, 0.5 * hu - 2.0 * hw) < 1e-5


def test_batched_hvp_weighting(sd, oracle):
    """Alg. 1: batches of sizes 1 and 3 == one concatenated 4-sample batch."""
    from paper_2505_11564_b200 import gpt
    cfg, S = TINY, 32
    tok, tgt = gpt.synthetic_tokens(cfg["vocab"], 4, S, 1, 0)
    whole = gpt.GptHvp(cfg, 4, S, init_seed=0, gain_scale=0.1, bias_scale=0.1, tokens=tok, targets=tgt)
    e1 = gpt.GptHvp(cfg, 1, S, theta=whole.theta, tokens=tok[:S], targets=tgt[:S])
    e3 = gpt.GptHvp(cfg, 3, S, theta=whole.theta, tokens=tok[S:], targets=tgt[S:])
    v = torch.tensor(oracle.draw_probe(whole.P, 9, 1, prec=0), dtype=torch.float32, device="cuda")
    a = whole.hvp(v).double().cpu().numpy()
    b = gpt.batched_hvp([e1, e3], v).double().cpu().numpy()
    assert rel(b, a) < 1e-6


def test_hvp_gpt2_small_dims_vs_torch_f64(sd):
    """Full GPT-2-small shapes (124M params, V=50257) at a short sequence,
    against float64 torch double-backward on the same device."""
    import torch_gpt
    from paper_2505_11564_b200 import gpt
    cfg, B, S = gpt.GPT2_SMALL, 1, 64
    eng = gpt.GptHvp(cfg, B, S, init_seed=0, gain_scale=0.05, bias_scale=0.02)
    g = torch.Generator(device="cuda").manual_seed(5)
    v = (torch.randint(0, 2, (eng.P,), device="cuda", generator=g).float() * 2 - 1) / np.sqrt(eng.P)
    hv = eng.hvp(v).double()
    tok = torch.tensor(eng._tok, device="cuda").long()
    tgt = torch.tensor(eng._tgt, device="cuda").long()
    ref = torch_gpt.hvp(cfg, eng.theta.double(), tok, tgt, B, S, v.double())
    e = float((hv - ref).norm() / ref.norm())
    print(f"GPT-2-small HVP rel-L2 vs torch f64: {e:.3e}")
    assert e < TOL


def test_c3_shape_runs_and_is_symmetric():
    # BASELINE C3 decoder shape (1.3B: 24L, d2048, ff8192, V50257, ctx2048, tied) at
    # 1 x 2048 tokens on one GPU: finite, symmetric u^T H w == w^T H u, linear
    from paper_2505_11564_b200 import gpt
    C3 = dict(n_layer=24, d=2048, n_head=16, ff=8192, vocab=50257, ctx=2048)
    eng = gpt.GptHvp(C3, 1, 2048)
    assert eng.P == 1315723264
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(eng.P, device="cuda", generator=g) * 1e-3
    w = torch.randn(eng.P, device="cuda", generator=g) * 1e-3
    hu, hw = eng.hvp(u), eng.hvp(w)
    assert bool(torch.isfinite(hu).all()) and bool(torch.isfinite(hw).all())
    a, b = float(torch.dot(hu.double(), w.double())), float(torch.dot(u.double(), hw.double()))
    assert abs(a - b) <= 1e-4 * max(abs(a), abs(b))
    hs = eng.hvp((0.5 * u - 2.0 * w).contiguous())
    lin = 0.5 * hu.double() - 2.0 * hw.double()
    assert float((hs.double() - lin).norm() / lin.norm()) < 1e-5
    eng.close()


LTINY = dict(n_layer=2, d=64, n_head=4, ff=96, vocab=96, ctx=32, arch=1, rope_base=10000)


def test_llama_layout_matches_oracle(sd, oracle):
    from paper_2505_11564_b200 import gpt
    for cfg in (LTINY, dict(LTINY, n_kv_head=2), gpt.LLAMA2_7B, gpt.LLAMA_70B):
        assert gpt.param_count(cfg) == oracle.gpt_param_count(cfg)
    assert gpt.param_count(gpt.LLAMA2_7B) == 6738415616  # Llama-2-7B parameter count
    assert gpt.param_count(gpt.LLAMA_70B) == 70553706496  # SURVEY C5 (R1-Distill-Llama-70B shape, GQA 64/8)
    assert gpt.param_layout(LTINY) == oracle.gpt_layout(LTINY)
    assert gpt.param_layout(dict(LTINY, n_kv_head=2)) == oracle.gpt_layout(dict(LTINY, n_kv_head=2))


@pytest.mark.parametrize("cfg,B,S", [(LTINY, 2, 32), (dict(LTINY, n_layer=1, n_head=2, d=32, ff=40), 3, 16),
                                     (dict(LTINY, n_kv_head=2), 2, 32), (dict(LTINY, n_head=8, d=64, n_kv_head=1), 1, 24)])
def test_llama_hvp_vs_oracle(sd, oracle, cfg, B, S):
    # Llama-style decoder (RMSNorm, RoPE, SwiGLU, untied head; BASELINE C4/C5 family)
    from paper_2505_11564_b200 import gpt
    eng = gpt.GptHvp(cfg, B, S, init_seed=0, gain_scale=0.1, bias_scale=0.1)
    th = eng.theta_numpy()
    assert np.array_equal(th, oracle.gpt_init(cfg, 0, 0.1, 0.1, prec=0))
    tok, tgt = eng.tokens_numpy()
    for seed in (3, 4):
        v = oracle.draw_probe(eng.P, seed, 1, prec=0)
        hv = eng.hvp_numpy(v)
        ref = oracle.gpt_hvp(cfg, th, tok, tgt, B, S, v)
        assert rel(hv, ref) < TOL, rel(hv, ref)
    assert abs(eng.loss() - oracle.gpt_loss(cfg, th, tok, tgt, B, S)) < 1e-5


def test_llama_finite_differences_and_symmetry(sd, oracle):
    from paper_2505_11564_b200 import gpt
    cfg, B, S = LTINY, 2, 32
    eng = gpt.GptHvp(cfg, B, S, init_seed=1, gain_scale=0.1)
    th = eng.theta_numpy()
    tok, tgt = eng.tokens_numpy()
    rng = np.random.default_rng(1)
    v = rng.standard_normal(eng.P).astype(np.float32).astype(np.float64)
    hv = eng.hvp_numpy(v)
    e = 1e-5
    fd = (oracle.gpt_grad(cfg, th + e * v, tok, tgt, B, S) - oracle.gpt_grad(cfg, th - e * v, tok, tgt, B, S)) / (2 * e)
    assert rel(hv, fd) < 2e-5
    u = rng.standard_normal(eng.P).astype(np.float32).astype(np.float64)
    hu = eng.hvp_numpy(u)
    assert abs(hu @ v - u @ hv) <= 1e-5 * np.linalg.norm(hu) * np.linalg.norm(v)


def test_llama2_7b_layer_shape_runs():
    # two decoder layers of the Llama-2-7B shape (d4096, ff11008, 32 heads, V32000)
    # at 1 x 1024 tokens: finite, symmetric Hv through the Lanczos-facing operator
    from paper_2505_11564_b200 import gpt
    cfg = dict(gpt.LLAMA2_7B, n_layer=2)
    eng = gpt.GptHvp(cfg, 1, 1024)
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(eng.P, device="cuda", generator=g) * 1e-3
    w = torch.randn(eng.P, device="cuda", generator=g) * 1e-3
    hu, hw = eng.hvp(u), eng.hvp(w)
    assert bool(torch.isfinite(hu).all()) and bool(torch.isfinite(hw).all())
    a, b = float(torch.dot(hu.double(), w.double())), float(torch.dot(u.double(), hw.double()))
    assert abs(a - b) <= 1e-4 * max(abs(a), abs(b))
    eng.close()


@pytest.mark.parametrize("cfg", [dict(LTINY, n_kv_head=2, bf16_weights=1), dict(TINY, bf16_weights=1)])
def test_bf16_weights_engine(sd, oracle, cfg):
    # BASELINE C5 "bf16 weights": bf16-valued parameters are exact in tf32, so the
    # engine keeps no weight residuals and runs the weight products with 2 MMAs.
    # Bit-identical to the residual engine on the same parameters; f64 oracle 1e-5.
    from paper_2505_11564_b200 import gpt
    B, S = 2, 32
    eng = gpt.GptHvp(cfg, B, S, init_seed=0, gain_scale=0.1, bias_scale=0.1)
    th = eng.theta
    assert bool(((th.view(torch.int32) & 0xFFFF) == 0).all())  # bf16-valued
    ref_cfg = dict(cfg, bf16_weights=0)
    eng32 = gpt.GptHvp(ref_cfg, B, S, theta=th.clone())
    assert eng.workspace.numel() < eng32.workspace.numel()  # no weight residuals
    v = torch.tensor(oracle.draw_probe(eng.P, 3, 1, prec=0), dtype=torch.float32, device="cuda")
    hv = eng.hvp(v)
    assert torch.equal(hv, eng32.hvp(v))
    tok, tgt = eng.tokens_numpy()
    ref = oracle.gpt_hvp(cfg, eng.theta_numpy(), tok, tgt, B, S, v.double().cpu().numpy())
    assert rel(hv.double().cpu().numpy(), ref) < TOL
    # non-bf16 parameters are refused
    with pytest.raises(sd.ConfigError):
        gpt.GptHvp(cfg, B, S, theta=th + 1e-3)


_AB_SCRIPT = r"""
import sys, hashlib
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2505_11564_b200 import gpt
cfg = dict(n_layer=2, d=64, n_head=4, ff=256, vocab=96, ctx=64)
eng = gpt.GptHvp(cfg, 8, 64, init_seed=2, gain_scale=0.1, bias_scale=0.1)
v = np.random.default_rng(7).standard_normal(eng.P).astype(np.float32).astype(np.float64)
hv = np.ascontiguousarray(eng.hvp_numpy(v))
print(hashlib.sha256(hv.tobytes()).hexdigest())
"""


def test_column_reduction_paths_bitwise(sd):
    """The 16-byte column reductions (k_colred4) sum every column in the scalar
    kernel's order (k_colred1, forced by SD_COLRED1=1): Hv is bit-identical.
    T = 512 token rows -> 8 row groups, so the ordered stage-2 fold runs."""
    import os, subprocess, sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    out = {}
    for tag, extra in (("vec", {}), ("scalar", {"SD_COLRED1": "1"})):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-c", _AB_SCRIPT, root], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = r.stdout.strip().splitlines()[-1]
    assert out["vec"] == out["scalar"], out


@pytest.mark.parametrize("cfg", [TINY, dict(LTINY, n_kv_head=2)])
def test_micro_batched_hvp_equals_whole_batch(sd, oracle, cfg):
    """PAPER.md Alg. 1 over a loader of micro-batches (h += u b): 4 micro-batches
    of 1 sequence == the 4-sequence batch (GPT-2 tied-head block and Llama);
    recomputation and on-chip probe residuals change no bit; vs the f64 oracle."""
    from paper_2505_11564_b200 import gpt
    S = 32
    tok, tgt = gpt.synthetic_tokens(cfg["vocab"], 4, S, seed=1)
    whole = gpt.GptHvp(cfg, 4, S, init_seed=0, gain_scale=0.1, bias_scale=0.1, tokens=tok, targets=tgt)
    mb = gpt.GptHvp(cfg, 1, S, theta=whole.theta, tokens=tok, targets=tgt, micro_batches=4)
    rc = gpt.GptHvp(cfg, 1, S, theta=whole.theta, tokens=tok, targets=tgt, micro_batches=4, recompute=True,
                    probe_residual=False)
    assert mb.workspace.numel() < whole.workspace.numel() and rc.workspace.numel() < mb.workspace.numel()
    v = torch.tensor(oracle.draw_probe(whole.P, 9, 1, prec=0), dtype=torch.float32, device="cuda")
    a, b, c = whole.hvp(v), mb.hvp(v), rc.hvp(v)
    assert torch.equal(b, c)
    assert float((b - a).norm() / a.norm()) < 3e-6  # fp32 sums over micro-batches vs within one batch
    ref = oracle.gpt_hvp(cfg, whole.theta_numpy(), tok.astype(np.uint32), tgt.astype(np.uint32), 4, S,
                         v.double().cpu().numpy())
    assert rel(b.double().cpu().numpy(), ref) < TOL
    assert abs(mb.loss() - whole.loss()) < 1e-6


def test_micro_batched_data_sharded_workers(sd):
    """C3's data-sharded HVP with micro-batches: 2 in-process workers, each 2
    micro-batches of 1 sequence, Lanczos vectors split between them (all-gather
    q, reduce-scatter Hv) == one worker with the whole 4-sequence batch."""
    from paper_2505_11564_b200 import gpt
    cfg = dict(n_layer=2, d=64, n_head=4, ff=128, vocab=96, ctx=32)
    B, S = 4, 32
    tok, tgt = gpt.synthetic_tokens(cfg["vocab"], B, S, seed=1)
    lc = sd.LanczosConfig(k_max=6, reorthogonalize=sd.REORTH_FULL, prec=sd.F32, reduction=sd.REDUCE_TREE,
                          probe=sd.ProbeSpec(seed=5, distribution=sd.RADEMACHER))
    whole = gpt.GptHvp(cfg, B, S, init_seed=0, gain_scale=0.1, tokens=tok, targets=tgt)
    a = sd.lanczos_run(whole.operator(), lc)
    lay = sd.split_evenly(whole.P, 2)

    def worker(r, comm):
        sl = slice(r * 2 * S, (r + 1) * 2 * S)
        e = gpt.GptHvp(cfg, 1, S, theta=whole.theta.clone(), tokens=tok[sl], targets=tgt[sl], micro_batches=2,
                       loss_scale=1.0 / (B * S))
        res = sd.lanczos_run(e.operator(comm, layout=lay), lc, layout=lay, comm=comm)
        e.close()
        return res

    out = sd.run_workers(2, worker)
    for r in out:
        assert np.max(np.abs(r.alphas - a.alphas)) <= 1e-5 * np.max(np.abs(a.alphas))


def test_c3_shape_micro_batched_recompute():
    # BASELINE C3 (1.3B GPT-2-architecture decoder) as it runs in bench.py
    # --workload c3: micro-batches of 1 x 2048 tokens with recomputation;
    # finite, symmetric, and the workspace of 2 micro-batches equals that of one
    from paper_2505_11564_b200 import gpt
    C3 = dict(n_layer=24, d=2048, n_head=16, ff=8192, vocab=50257, ctx=2048)
    eng = gpt.GptHvp(C3, 1, 2048, micro_batches=2, recompute=True)
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(eng.P, device="cuda", generator=g) * 1e-3
    w = torch.randn(eng.P, device="cuda", generator=g) * 1e-3
    hu, hw = eng.hvp(u), eng.hvp(w)
    assert bool(torch.isfinite(hu).all()) and bool(torch.isfinite(hw).all())
    a, b = float(torch.dot(hu.double(), w.double())), float(torch.dot(u.double(), hw.double()))
    assert abs(a - b) <= 1e-4 * max(abs(a), abs(b))
    assert eng.workspace.numel() < 40e9
    eng.close()
