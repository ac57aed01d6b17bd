"""Llama-2-7B layer shape (BASELINE C4 family) on one GPU: HVP timing for L
layers at B x S tokens (random init, synthetic tokens)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B, S = 1, int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = dict(gpt.LLAMA2_7B, n_layer=L)
eng = gpt.GptHvp(cfg, B, S)
v = torch.randn(eng.P, device="cuda") / 1e3
out = torch.empty_like(v)
eng.hvp(v, out); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3): eng.hvp(v, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
d, ff, V, T, H = 4096, 11008, 32000, B * S, 32
nmm = L * (4 * d * d + 3 * d * ff) + V * d   # qkv+o, gate+up+down, output head
fl = 16 * nmm * T + 36 * L * B * H * S * S * (d // H)
print(f"llama2-7b x{L} layers, {T} tokens: P={eng.P} HVP {ms:.1f} ms  {fl / ms / 1e9:.1f} TF/s algorithmic "
      f"({fl / 1e12:.1f} TFLOP) finite={bool(torch.isfinite(out).all())}")
