"""BASELINE configs[2] (C3) shape, 1.3B GPT-2-architecture decoder, one
2048-token sequence (optionally as micro-batches): device HVP vs float64 torch
double-backward (tests/torch_gpt.py).

    python tools/c3_parity.py [--layers 24] [--seq 2048] [--micro-batches 1]
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

import torch_gpt  # noqa: E402
from paper_2505_11564_b200 import gpt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=24)
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--micro-batches", type=int, default=1)
a = ap.parse_args()
cfg = dict(n_layer=a.layers, d=2048, n_head=16, ff=8192, vocab=50257, ctx=2048)
B, S = a.batch * a.micro_batches, a.seq
eng = gpt.GptHvp(cfg, a.batch, S, init_seed=0, gain_scale=0.05, bias_scale=0.02, micro_batches=a.micro_batches)
g = torch.Generator(device="cuda").manual_seed(5)
v = ((torch.randint(0, 2, (eng.P,), device="cuda", generator=g).float() * 2 - 1) / np.sqrt(eng.P)).contiguous()
hv = eng.hvp(v).double().cpu()
theta = eng.theta.double()
tok = torch.tensor(eng._tok, device="cuda").long()
tgt = torch.tensor(eng._tgt, device="cuda").long()
eng.close()
del eng
torch.cuda.empty_cache()
ref = torch_gpt.hvp(cfg, theta, tok, tgt, B, S, v.double()).cpu()
print(json.dumps({"config": f"C3 shape, {a.layers} layers, {B} x {S} tokens, {a.micro_batches} micro-batches",
                  "params": int(theta.numel()), "hvp_rel_l2": float((hv - ref).norm() / ref.norm()),
                  "peak_gb": torch.cuda.max_memory_allocated() / 1e9}))
