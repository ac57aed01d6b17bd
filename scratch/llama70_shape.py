"""R1-Distill-Llama-70B layer shape (BASELINE C5 family: d8192, ff28672,
V128256, GQA 64/8) on one GPU: HVP timing for L layers at B x S tokens."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
cfg = dict(gpt.LLAMA_70B, n_layer=L)
eng = gpt.GptHvp(cfg, 1, S)
v = torch.randn(eng.P, device="cuda") / 1e3
out = torch.empty_like(v)
eng.hvp(v, out); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3): eng.hvp(v, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
d, ff, V, H, KVd = 8192, 28672, 128256, 64, 1024
nmm = L * (d * (d + 2 * KVd) + d * d + 3 * d * ff) + V * d
fl = 16 * nmm * S + 36 * L * H * S * S * (d // H)
print(f"llama-70b x{L} layers, {S} tokens: P={eng.P} HVP {ms:.1f} ms  {fl / ms / 1e9:.1f} TF/s algorithmic "
      f"({fl / 1e12:.1f} TFLOP) finite={bool(torch.isfinite(out).all())}")
