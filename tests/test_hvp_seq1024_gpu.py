"""HVP parity at the benchmark's own shapes (BASELINE configs[1]: GPT-2-small,
8 x 1024 tokens) and at S >= 1024 for the Llama-style engine with grouped-query
attention, against float64 torch double-backward (tests/torch_gpt.py, itself
pinned to the C++ oracle in tests/test_oracle.py). These shapes exercise what
the S <= 64 oracle comparisons cannot reach: the triangular causal tile walk
and K-range trimming of the attention products, the register-resident softmax
R-op kernels (S % 128 == 0), and the T = 8192 split-K choices.

Tolerance (north star): rel-L2 <= 1e-5 against the f64 reference.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def gpt():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2505_11564_b200 import gpt
    return gpt


def _rademacher(P, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return ((torch.randint(0, 2, (P,), device="cuda", generator=g).float() * 2 - 1) / np.sqrt(P)).contiguous()


def _engine_vs_torch(gpt, cfg, B, S, **init):
    import torch_gpt
    eng = gpt.GptHvp(cfg, B, S, **init)
    v = _rademacher(eng.P, 5)
    hv = eng.hvp(v).double().cpu()
    theta = eng.theta.double()
    tok = torch.tensor(eng._tok, device="cuda").long()
    tgt = torch.tensor(eng._tgt, device="cuda").long()
    eng.close()
    del eng
    torch.cuda.empty_cache()
    ref = torch_gpt.any_hvp(cfg, theta, tok, tgt, B, S, v.double()).cpu()
    del theta
    torch.cuda.empty_cache()
    return float((hv - ref).norm() / ref.norm())


@pytest.mark.parametrize("B", [1, 2, 8])
def test_gpt2_small_seq1024_vs_torch_f64(gpt, B):
    """The bench model at S = 1024 (B = 8 is the bench batch itself), the
    bench's own init (seed 0, unit LN gains, zero biases)."""
    e = _engine_vs_torch(gpt, gpt.GPT2_SMALL, B, 1024, init_seed=0)
    print(f"GPT-2-small B={B} S=1024 HVP rel-L2 vs torch f64: {e:.3e}")
    assert e < TOL


@pytest.mark.parametrize("S", [128, 1024])
def test_gpt2_width_two_layers_vs_torch_f64(gpt, S):
    # perturbed LN gains/biases so every second-order LN term is live
    cfg = dict(gpt.GPT2_SMALL, n_layer=2)
    e = _engine_vs_torch(gpt, cfg, 2, S, init_seed=3, gain_scale=0.1, bias_scale=0.05)
    print(f"GPT-2 width, 2 layers, S={S}: {e:.3e}")
    assert e < TOL


@pytest.mark.parametrize("cfg,B,S", [
    # grouped-query attention (16 query heads on 4 kv heads) at S = 1024
    (dict(n_layer=2, d=1024, n_head=16, n_kv_head=4, ff=2816, vocab=32000, ctx=2048, arch=1, rope_base=10000), 2, 1024),
    # GQA 8:1 (the C5 ratio) at S = 2048
    (dict(n_layer=1, d=1024, n_head=16, n_kv_head=2, ff=2816, vocab=32000, ctx=4096, arch=1, rope_base=500000), 1, 2048),
    # one layer of the Llama-2-7B shape (C4), MHA, S = 1024
    (dict(n_layer=1, d=4096, n_head=32, ff=11008, vocab=32000, ctx=4096, arch=1, rope_base=10000), 1, 1024),
])
def test_llama_long_sequence_vs_torch_f64(gpt, cfg, B, S):
    e = _engine_vs_torch(gpt, cfg, B, S, init_seed=1, gain_scale=0.1)
    print(f"Llama {cfg['d']}/{cfg['n_head']}/{cfg.get('n_kv_head', 0)} B={B} S={S}: {e:.3e}")
    assert e < TOL


_DIGEST = r"""
import sys, hashlib
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from paper_2505_11564_b200 import gpt
cfg = dict(gpt.GPT2_SMALL, n_layer=2)
eng = gpt.GptHvp(cfg, 2, 1024, init_seed=2, gain_scale=0.1, bias_scale=0.1)
g = torch.Generator(device="cuda").manual_seed(7)
v = torch.randn(eng.P, device="cuda", generator=g).contiguous()
hv = eng.hvp(v).cpu().numpy()
print(hashlib.sha256(hv.tobytes()).hexdigest())
"""


def test_pdl_on_off_bitwise(gpt):
    """Programmatic dependent launch (GEMMs and their secondaries, incl. the
    register softmax R-op at S % 128 == 0) changes only launch overlap, never
    a bit of Hv: SD_GEMM_PDL=0 vs the default, in fresh processes."""
    out = {}
    for tag, extra in (("pdl", {}), ("nopdl", {"SD_GEMM_PDL": "0"})):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-c", _DIGEST, str(ROOT)], env=env, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = r.stdout.strip().splitlines()[-1]
    assert out["pdl"] == out["nopdl"], out


@pytest.mark.parametrize("micro_batches", [1, 2])
def test_c3_width_vs_torch_f64(gpt, micro_batches):
    """BASELINE configs[2] width (d 2048, 16 heads of 128, ff 8192, V 50257) at
    S = 2048 with 4 of its 24 layers, whole or as micro-batches (the full
    24-layer model gives 5.9e-6 / 6.1e-6 with tools/c3_parity.py, at 170 GB of
    f64 reference memory: profiles/r02_c3_parity_full.json)."""
    cfg = dict(n_layer=4, d=2048, n_head=16, ff=8192, vocab=50257, ctx=2048)
    S = 2048 if micro_batches == 1 else 1024
    import torch_gpt
    eng = gpt.GptHvp(cfg, 1, S, init_seed=0, gain_scale=0.05, bias_scale=0.02, micro_batches=micro_batches)
    v = _rademacher(eng.P, 5)
    hv = eng.hvp(v).double().cpu()
    theta = eng.theta.double()
    tok = torch.tensor(eng._tok, device="cuda").long()
    tgt = torch.tensor(eng._tgt, device="cuda").long()
    B = eng.B
    eng.close()
    del eng
    torch.cuda.empty_cache()
    ref = torch_gpt.hvp(cfg, theta, tok, tgt, B, S, v.double()).cpu()
    e = float((hv - ref).norm() / ref.norm())
    print(f"C3 width, 4 layers, {B} x {S}: {e:.3e}")
    assert e < TOL


_GRAPH = r"""
import sys, hashlib, json
import torch
sys.path.insert(0, sys.argv[1])
from paper_2505_11564_b200 import gpt
from paper_2505_11564_b200._lib import lib
cfg = dict(gpt.GPT2_SMALL, n_layer=2)
eng = gpt.GptHvp(cfg, 2, 1024, init_seed=2, gain_scale=0.1, bias_scale=0.1)
out = torch.empty(eng.P, device="cuda")
g = torch.Generator(device="cuda").manual_seed(7)
res = []
def call(v):
    n0 = lib().sd_launch_count()
    eng.hvp(v, out)
    torch.cuda.synchronize()
    res.append([hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest(), lib().sd_launch_count() - n0])
for i in range(4):  # eager warm-up, capture, replay, replay (fixed output pointer)
    call(torch.randn(eng.P, device="cuda", generator=g).contiguous())
# a new batch (same loss scale: replayed with the new token contents), then a
# new loss scale (a captured kernel argument: eager, recapture, replay)
tok, tgt = gpt.synthetic_tokens(cfg["vocab"], 2, 1024, seed=9)
eng.set_batch(tok, tgt)
v = torch.randn(eng.P, device="cuda", generator=g).contiguous()
call(v)
eng.set_batch(tok, tgt, loss_scale=0.25 / 2048)
for i in range(3):
    call(v)
print(json.dumps(res))
"""


def test_cuda_graph_replay_bitwise(gpt):
    """The whole-model HVP is captured into a CUDA graph at its second call with
    the same output pointer and replayed afterwards: Hv of every call equals
    the always-eager run (SD_GPT_GRAPH=0) bitwise, and every call reports the
    same number of kernel launches (replays count the graph's kernels)."""
    import json
    out = {}
    for tag, extra in (("graph", {}), ("eager", {"SD_GPT_GRAPH": "0"})):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-c", _GRAPH, str(ROOT)], env=env, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = json.loads(r.stdout.strip().splitlines()[-1])
    assert [h for h, _ in out["graph"]] == [h for h, _ in out["eager"]]
    counts = [n for _, n in out["graph"]] + [n for _, n in out["eager"]]
    assert len(set(counts)) == 1 and counts[0] > 0, counts


_HV_NPY = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from paper_2505_11564_b200 import gpt
eng = gpt.GptHvp(gpt.GPT2_SMALL, 4, 1024, init_seed=4, gain_scale=0.1, bias_scale=0.1)
g = torch.Generator(device="cuda").manual_seed(3)
v = torch.randn(eng.P, device="cuda", generator=g).contiguous()
np.save(sys.argv[2], eng.hvp(v).cpu().numpy())
"""


def test_twin_products_match_two_launches(gpt, tmp_path):
    """Twin launches (a weight's primal and tangent products in one launch,
    the score products S / dS and gP / gdP likewise) against the two-launch
    path (SD_GEMM_TWIN=0) on GPT-2-small at 4 x 1024 tokens: identical where
    the split counts agree, else the same sums in another split partition --
    within 2e-6 (the parity tests above bound both against float64)."""
    import numpy as np
    out = {}
    for tag, extra in (("twin", {}), ("two", {"SD_GEMM_TWIN": "0"})):
        f = tmp_path / f"{tag}.npy"
        r = subprocess.run([sys.executable, "-c", _HV_NPY, str(ROOT), str(f)], env=dict(os.environ, **extra),
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = np.load(f).astype(np.float64)
    e = float(np.linalg.norm(out["twin"] - out["two"]) / np.linalg.norm(out["two"]))
    print(f"twin vs two launches: {e:.3e}")  # 5.1e-7 on the B200
    assert e < 2e-6

