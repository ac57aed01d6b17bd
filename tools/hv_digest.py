"""Hv digest of the GPT-2-small HVP at the bench shape (8 x 1024 tokens): for
bitwise A/B checks of launch-order / walk changes (SD_GEMM_MFAST=0/1,
SD_GEMM_PDL=0/1) and the HVP's median time over a few repetitions.

    python tools/hv_digest.py [--batch 8] [--reps 5]
"""
import argparse
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_11564_b200 import gpt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--seq", type=int, default=1024)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
eng = gpt.GptHvp(gpt.GPT2_SMALL, a.batch, a.seq, init_seed=0)
g = torch.Generator(device="cuda").manual_seed(7)
v = torch.randn(eng.P, device="cuda", generator=g).contiguous()
hv = eng.hvp(v)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.hvp(v, hv)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"digest": hashlib.sha256(hv.cpu().numpy().tobytes()).hexdigest()[:16],
                  "hvp_ms_median": float(np.median(ts)), "hvp_ms": ts}))
