"""HVP time of the Llama-2-7B-shaped stage (4 layers, 1 x 1024 tokens and 2 x 2048) with f32 weights
(3 MMAs per weight product + weight residuals) vs bf16-valued weights (2 MMAs, no residuals)."""
import sys, json
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
res = []
for (B, S) in ((1, 1024), (2, 2048)):
    for bf in (0, 1):
        cfg = dict(gpt.LLAMA2_7B, n_layer=4, bf16_weights=bf)
        eng = gpt.GptHvp(cfg, B, S, init_seed=0)
        v = torch.randn(eng.P, device="cuda") * 1e-3
        out = torch.empty_like(v)
        for _ in range(2): eng.hvp(v, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5): eng.hvp(v, out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        r = {"tokens": B * S, "bf16_weights": bf, "ms": ms, "workspace_gb": eng.workspace.numel() / 1e9}
        print(r, flush=True); res.append(r)
        eng.close(); del eng, v, out; torch.cuda.empty_cache()
print(json.dumps(res))
