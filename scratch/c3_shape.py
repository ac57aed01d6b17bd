"""C3 shape (1.3B GPT decoder: 24L, d2048, ff8192, V50257, ctx2048, tied) on one
GPU: batch 1 x 2048 tokens, HVP timing and a few Lanczos steps."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2505_11564_b200 as sd
from paper_2505_11564_b200 import gpt
C3 = dict(n_layer=24, d=2048, n_head=16, ff=8192, vocab=50257, ctx=2048)
B, S = int(sys.argv[1]) if len(sys.argv) > 1 else 1, 2048
eng = gpt.GptHvp(C3, B, S)
print("P", eng.P, "workspace GB", eng.workspace.numel() / 1e9)
v = torch.randn(eng.P, device="cuda") / 1e3
out = torch.empty_like(v)
eng.hvp(v, out); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3): eng.hvp(v, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
L, d, ff, V, T = 24, 2048, 8192, 50257, B * S
nmm = L * 12 * d * d + V * d
fl = 16 * nmm * T + 36 * L * B * 16 * S * S * (d // 16)
print(f"HVP {ms:.1f} ms  {fl / ms / 1e9:.1f} TF/s algorithmic ({fl / 1e12:.1f} TFLOP)  finite={bool(torch.isfinite(out).all())}")
cfg = sd.LanczosConfig(k_max=10, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                       probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
t0 = time.time()
res = sd.lanczos_run(eng.operator(), cfg)
print("lanczos 10 steps", time.time() - t0, "s; alphas", res.alphas[:4], "betas", res.betas[:3])
