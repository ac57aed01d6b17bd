"""One Lanczos step of the bench workload (GPT-2-small, 8 x 1024 tokens, full
reorth, tree reductions) at reorth width j, inside an NVTX range "step" so
that ncu captures exactly that step's launch list:

    ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,\
        dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file launches.csv python tools/one_step.py --j 50
    python tools/summarize_launches.py launches.csv profiles/<name>.md profiles/<name>.json
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2505_11564_b200 as sd  # noqa: E402
from paper_2505_11564_b200 import gpt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--j", type=int, default=50)
ap.add_argument("--reduction", default="tree", choices=["tree", "ordered"])
a = ap.parse_args()
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024, init_seed=0)
cfg = sd.LanczosConfig(k_max=100, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                       reduction=sd.REDUCE_TREE if a.reduction == "tree" else sd.REDUCE_ORDERED,
                       probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
L = sd.Lanczos(eng.operator(), cfg)
for _ in range(a.j - 1):
    L.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
L.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("alphas", L.result().alphas.size)
