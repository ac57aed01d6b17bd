"""Lanczos-engine microbenchmark (no HVP): a diagonal operator of the
GPT-2-small size drives the device engine; per-step times of the recurrence
+ reorthogonalisation in ordered and tree mode around reorth width j.

    python tools/lanczos_kernels.py [--P 124439808] [--j 50] [--modes tree,ordered]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2505_11564_b200 as sd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=124439808)
ap.add_argument("--j", type=int, default=50)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--modes", default="tree,ordered")
a = ap.parse_args()
d = torch.linspace(-3.0, 5.0, a.P, device="cuda")
op = sd.diag_operator(d)
for mode in a.modes.split(","):
    red = sd.REDUCE_TREE if mode == "tree" else sd.REDUCE_ORDERED
    cfg = sd.LanczosConfig(k_max=a.j + a.steps + 2, reorthogonalize=sd.REORTH_FULL, prec=sd.F32, reduction=red,
                           probe=sd.ProbeSpec(seed=1, distribution=sd.RADEMACHER))
    L = sd.Lanczos(op, cfg)
    for _ in range(a.j - 1):
        L.step()
    r0 = L.result()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        L.step()
    e1.record()
    torch.cuda.synchronize()
    r1 = L.result()
    ms = e0.elapsed_time(e1) / a.steps
    jm = a.j + (a.steps - 1) / 2
    byt = 4.0 * a.P * ((3 * jm + 8) if mode == "tree" else (7 + 3 * jm))
    print(json.dumps({"mode": mode, "P": a.P, "j_mean": jm, "ms_per_step": ms,
                      "recurrence_ms": (r1.ms_recurrence - r0.ms_recurrence) / a.steps,
                      "reorth_ms": (r1.ms_reorth - r0.ms_reorth) / a.steps,
                      "apply_ms": (r1.ms_apply - r0.ms_apply) / a.steps,
                      "algorithmic_GBps": byt / (ms * 1e-3) / 1e9}), flush=True)
    L.close()
