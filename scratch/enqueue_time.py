"""CPU enqueue time of one HVP / one Lanczos step vs its GPU time."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2505_11564_b200 as sd
from paper_2505_11564_b200 import gpt
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024)
v = torch.randn(eng.P, device="cuda") / 1e4
out = torch.empty_like(v)
for _ in range(3): eng.hvp(v, out)
torch.cuda.synchronize()
for _ in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter(); e0.record(); eng.hvp(v, out); e1.record(); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"hvp: enqueue {1e3*(t1-t0):.2f} ms, gpu {e0.elapsed_time(e1):.2f} ms, wall {1e3*(t2-t0):.2f} ms")
cfg = sd.LanczosConfig(k_max=100, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                       probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
L = sd.Lanczos(eng.operator(), cfg)
for _ in range(45): L.step()
torch.cuda.synchronize()
for _ in range(5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter(); e0.record(); L.step(); e1.record(); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"step: call {1e3*(t1-t0):.2f} ms, gpu {e0.elapsed_time(e1):.2f} ms, wall {1e3*(t2-t0):.2f} ms")
