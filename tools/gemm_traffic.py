"""GEMM traffic of one GPT-2-small HVP at the bench shape (8 x 1024 tokens).

Step 1 (plain run): every GEMM launch of one HVP is recorded with its shape
(sd_gemm_profile_dump); the ALGORITHMIC bytes of a launch are
4 * batch * (nsrc * (M*K + N*K) + M*N) -- each operand read once, C written
once (tf32 residual arrays are implementation traffic, not algorithmic).

Step 2 (under ncu): run with --ncu and the launches of the same HVP are
captured by
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
        -k regex:k_gemm --csv --log-file <csv> python tools/gemm_traffic.py --ncu
and `--summarise <csv>` writes profiles/<out>.json with the measured DRAM
bytes per launch next to the algorithmic bytes per launch (bench.py reports
both as roofline.traffic / roofline.algorithmic_bytes).
"""
import argparse
import csv
import ctypes as C
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true", help="run one HVP only (the ncu pass)")
ap.add_argument("--summarise", default=None, help="ncu csv log to summarise")
ap.add_argument("--shapes", default=str(ROOT / "gpurun_out" / "gemm_shapes.csv"))
ap.add_argument("--out", default=str(ROOT / "profiles" / "gemm_traffic.json"))
ap.add_argument("--batch", type=int, default=8, help="sequences of 1024 tokens (8 = the bench; 1 = one rank at N = 8)")
a = ap.parse_args()

if a.summarise:
    rows = [r for r in csv.reader(open(a.summarise)) if len(r) > 10]
    h = rows[0]
    by = defaultdict(dict)
    for r in rows[1:]:
        by[r[h.index("ID")]][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
        by[r[h.index("ID")]]["name"] = r[h.index("Kernel Name")]
    gem = [v for v in by.values() if "k_gemm" in v["name"]]
    rd = sum(v["dram__bytes_read.sum"] for v in gem)
    wr = sum(v["dram__bytes_write.sum"] for v in gem)
    shp = list(csv.DictReader(open(a.shapes)))
    alg = 0.0
    for s in shp:
        M, N, K, Z = (int(float(s[k])) for k in ("M", "N", "K", "batch"))
        if s["nsrc"] == "split":  # [A B | A B2 + A2 B]: A, A2 once, B | B2 (N wide) once, C | C2
            alg += 4.0 * Z * (2 * M * K + N * K + M * N)
        elif s["nsrc"] == "twin":  # A B and A2 B + A B2: A, A2, B, B2 once, C and C2
            alg += 4.0 * Z * (2 * M * K + 2 * N * K + 2 * M * N)
        else:
            ns = int(float(s["nsrc"]))
            alg += 4.0 * Z * (ns * (M * K + N * K) + M * N)
    out = {"launches_ncu": len(gem), "launches_shapes": len(shp),
           "bytes_per_launch": (rd + wr) / max(1, len(gem)), "dram_read_bytes": rd, "dram_write_bytes": wr,
           "algorithmic_bytes_per_launch": alg / max(1, len(shp)),
           "ratio_measured_over_algorithmic": (rd + wr) / alg if alg else None,
           "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every k_gemm* launch of one "
                  "GPT-2-small HVP (8x1024 tokens); algorithmic = 4*batch*(nsrc*(MK+NK)+MN) per launch "
                  "(each operand read once, each output written once; split pairs and twin products count "
                  "their distinct operands and both outputs)"}
    Path(a.out).write_text(json.dumps(out, indent=1))
    print(json.dumps(out))
    sys.exit(0)

import torch  # noqa: E402

from paper_2505_11564_b200 import gpt  # noqa: E402
from paper_2505_11564_b200._lib import check, lib  # noqa: E402

eng = gpt.GptHvp(gpt.GPT2_SMALL, a.batch, 1024, init_seed=0)
v = torch.randn(eng.P, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7)).contiguous()
if a.ncu:
    eng.hvp(v)
    torch.cuda.synchronize()
    sys.exit(0)
eng.hvp(v)
torch.cuda.synchronize()
L = lib()
check(L.sd_gemm_profile_begin())
eng.hvp(v)
torch.cuda.synchronize()
ms, fl, n = C.c_double(), C.c_double(), C.c_uint64()
check(L.sd_gemm_profile_end(C.byref(ms), C.byref(fl), C.byref(n)))
L.sd_gemm_profile_dump.argtypes = [C.c_char_p]
Path(a.shapes).parent.mkdir(exist_ok=True)
check(L.sd_gemm_profile_dump(a.shapes.encode()))
print(json.dumps({"gemm_ms": ms.value, "tflop": fl.value / 1e12, "launches": n.value}))
