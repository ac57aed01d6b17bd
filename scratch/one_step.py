"""One Lanczos step of the bench workload at column ~50 inside a
cudaProfilerStart/Stop window (for ncu --profile-from-start off)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2505_11564_b200 as sd
from paper_2505_11564_b200 import gpt
adv = int(sys.argv[1]) if len(sys.argv) > 1 else 50
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024)
cfg = sd.LanczosConfig(k_max=100, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                       probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
L = sd.Lanczos(eng.operator(), cfg)
for _ in range(adv):
    L.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
L.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", L.result().alphas.size)
