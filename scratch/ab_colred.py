"""A/B of the column reductions: run with SD_COLRED1=1 (scalar k_colred1) and
without (16-byte k_colred4); saves Hv for a bitwise comparison and prints the
HVP time (CUDA events, median of 10)."""
import sys, os
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
tag = sys.argv[1]
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024)
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.randn(eng.P, device="cuda", generator=g) / 1e3
out = torch.empty_like(v)
for _ in range(3): eng.hvp(v, out)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); eng.hvp(v, out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
bits = out.view(torch.int32).to(torch.int64)
digest = int(((bits * torch.arange(1, bits.numel() + 1, device="cuda", dtype=torch.int64) % 1000003)).sum().item())
print(tag, "digest", digest, "norm", out.double().norm().item())
print(tag, "hvp ms median", ts[5], "min", ts[0])
