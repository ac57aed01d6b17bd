"""One layer of the BASELINE C5 architecture (R1-Distill-Llama-70B shape: d8192,
ff28672, V128256, GQA 64/8, bf16-valued weights) at B x S tokens: device HVP
(bf16-weights engine, 2-MMA weight products) vs float64 torch double-backward,
then a k-step full-reorth Lanczos on both (device tree mode vs a float64 torch
Lanczos over the torch HVP): alpha/beta, Ritz values and weights.

    python tools/llama70_layer_parity.py [--seq 128] [--k 8]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_11564_b200 as sd  # noqa: E402
import torch_gpt  # noqa: E402
from paper_2505_11564_b200 import gpt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=128)
ap.add_argument("--k", type=int, default=5)
a = ap.parse_args()
cfg = dict(gpt.LLAMA_70B, n_layer=1, bf16_weights=1)
B, S, k = 1, a.seq, a.k
eng = gpt.GptHvp(cfg, B, S, init_seed=0, gain_scale=0.1)
P = eng.P
g = torch.Generator(device="cuda").manual_seed(3)
v = ((torch.randint(0, 2, (P,), device="cuda", generator=g).float() * 2 - 1) / np.sqrt(P)).contiguous()
hv = eng.hvp(v).double().cpu()
lc = sd.LanczosConfig(k_max=k, reorthogonalize=sd.REORTH_FULL, prec=sd.F32, reduction=sd.REDUCE_TREE,
                      probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
dev = sd.lanczos_run(eng.operator(), lc)
pool = sd.make_pool(P, 1)
q0 = torch.tensor(sd.gather(pool, sd.draw_probe(pool, lc.probe, sd.F32)), dtype=torch.float64)
theta = eng.theta.double()
tok = torch.tensor(eng._tok.astype(np.int64))
tgt = torch.tensor(eng._tgt.astype(np.int64))
eng.close()
del eng, pool
torch.cuda.empty_cache()
th = theta
tokd, tgtd = tok.cuda(), tgt.cuda()


def H(x):
    return torch_gpt.llama_hvp(cfg, th, tokd, tgtd, B, S, x)


def dot(x, y, chunk=1 << 27):  # f64 dots in chunks (cuBLAS dot takes int32 lengths; P = 2.96e9)
    return sum(float(x[i:i + chunk].double() @ y[i:i + chunk].double()) for i in range(0, x.numel(), chunk))


ref = H(v.double()).cpu()
hv_rel = float(((hv - ref).double().pow(2).sum() / ref.double().pow(2).sum()) ** 0.5)
# float64 Lanczos (full reorth = 2x CGS) over the torch HVP;
# the residual in f64 and the basis (rounded to f32, 12 GB a column) in host
# memory, each HVP input uploaded in f64
del v
torch.cuda.empty_cache()
Q = [q0.float()]
al, be = [], []
for j in range(k):
    r = H(Q[-1].cuda().double()).cpu()
    if j > 0:
        r -= be[-1] * Q[-2].double()
    alpha = dot(Q[-1], r)
    r -= alpha * Q[-1].double()
    for _ in range(2):
        c = [dot(qq, r) for qq in Q]
        for ci, qq in zip(c, Q):
            r -= ci * qq.double()
    beta = dot(r, r) ** 0.5
    al.append(alpha)
    if j + 1 == k:
        break
    be.append(beta)
    Q.append((r / beta).float())
    del r
tnorm = max(max(abs(x) for x in al), max(be))
rd = sd.ritz_decompose(dev.alphas, dev.betas)
rr = sd.ritz_decompose(np.array(al), np.array(be))
out = {"config": "LLAMA_70B shape, 1 layer, bf16 weights", "params": P, "tokens": B * S, "hvp_rel_l2": hv_rel,
       "alpha_beta_rel": float(max(np.max(np.abs(dev.alphas - al)), np.max(np.abs(dev.betas - be))) / tnorm),
       "ritz_values_rel": float(np.max(np.abs(rd.values - rr.values)) / (rr.values[-1] - rr.values[0])),
       "ritz_weights_abs": float(np.max(np.abs(rd.weights - rr.weights))),
       "peak_gb": torch.cuda.max_memory_allocated() / 1e9}
print(json.dumps(out))
