"""Eager vs CUDA-graph-replayed HVP at the bench shape (8 x 1024 tokens): the
engine captures its whole-model HVP at the second call with the same output
pointer (SD_GPT_GRAPH, default on). Runs both modes in fresh processes,
interleaved, and prints each call's median time and the Hv digest.

    python tools/graph_ab.py [--reps 10] [--rounds 2]
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

_CHILD = r"""
import hashlib, json, sys
import torch
sys.path.insert(0, sys.argv[1])
from paper_2505_11564_b200 import gpt
reps = int(sys.argv[2])
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024, init_seed=0)
g = torch.Generator(device="cuda").manual_seed(7)
v = torch.randn(eng.P, device="cuda", generator=g).contiguous()
out = torch.empty(eng.P, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):  # warm-up, capture, first replay
    eng.hvp(v, out)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    eng.hvp(v, out)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(json.dumps({"ms": ts[len(ts) // 2], "digest": hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]}))
"""

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--rounds", type=int, default=2)
a = ap.parse_args()
res = {"graph": [], "eager": []}
for _ in range(a.rounds):
    for tag, extra in (("graph", {}), ("eager", {"SD_GPT_GRAPH": "0"})):
        r = subprocess.run([sys.executable, "-c", _CHILD, str(ROOT), str(a.reps)], env=dict(os.environ, **extra),
                           capture_output=True, text=True, check=True)
        res[tag].append(json.loads(r.stdout.strip().splitlines()[-1]))
print(json.dumps(res))
