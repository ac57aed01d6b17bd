"""One GPT-2-small HVP (8 x 1024 tokens) after two warm-up HVPs, inside a profiler window."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024)
v = torch.randn(eng.P, device="cuda") / 1e4
out = torch.empty_like(v)
for _ in range(2): eng.hvp(v, out)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.hvp(v, out)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
