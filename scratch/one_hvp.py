import sys
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024)
v = torch.randn(eng.P, device="cuda") / 1e4
out = torch.empty_like(v)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    eng.hvp(v, out)
torch.cuda.synchronize()
print("ok")
