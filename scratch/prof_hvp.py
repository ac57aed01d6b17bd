import sys, ctypes as C, collections
sys.path.insert(0, '.')
import torch
import paper_2505_11564_b200 as sd
from paper_2505_11564_b200 import gpt
from paper_2505_11564_b200._lib import lib, check
L = lib()
eng = gpt.GptHvp(gpt.GPT2_SMALL, 8, 1024)
v = torch.randn(eng.P, device="cuda") / 1e4
out = torch.empty_like(v)
for _ in range(2): eng.hvp(v, out)
torch.cuda.synchronize()
check(L.sd_gemm_profile_begin())
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); eng.hvp(v, out); e1.record(); torch.cuda.synchronize()
ms, fl, n = C.c_double(), C.c_double(), C.c_uint64()
check(L.sd_gemm_profile_end(C.byref(ms), C.byref(fl), C.byref(n)))
L.sd_gemm_profile_dump.argtypes = [C.c_char_p]
check(L.sd_gemm_profile_dump(b"gpurun_out/gemm_prof.csv"))
print("hvp ms", e0.elapsed_time(e1), "gemm ms", ms.value, "TF/s", fl.value / ms.value / 1e9, "launches", n.value)
import csv
rows = list(csv.DictReader(open("gpurun_out/gemm_prof.csv")))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    k = (r["M"], r["N"], r["K"], r["batch"], r["a_mn"], r["b_mn"], r["causal"], r["splits"], r["nsrc"])
    agg[k][0] += 1; agg[k][1] += float(r["ms"]); agg[k][2] += float(r["flops"])
for k, (c, t, f) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:8.3f} ms {c:4d}x  {f / t / 1e9:7.1f} TF/s  M,N,K,batch,amn,bmn,causal,splits,nsrc={','.join(k)}")
