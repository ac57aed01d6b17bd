"""HVP time and GEMM breakdown of GPT-2-small at a per-rank batch of B sequences
(the strong-scaling shards of the 8 x 1024 bench batch: B = 8 / N)."""
import sys, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
from paper_2505_11564_b200._lib import lib, check
L = lib()
for B in (8, 4, 2, 1):
    eng = gpt.GptHvp(gpt.GPT2_SMALL, B, 1024, loss_scale=1.0 / 8192)
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
    check(L.sd_gemm_profile_dump(f"gpurun_out/gemm_prof_b{B}.csv".encode()))
    print(f"B={B}: hvp {e0.elapsed_time(e1):.2f} ms (x{8 // B} = {e0.elapsed_time(e1) * 8 / B:.1f}), gemm {ms.value:.2f} ms at {fl.value / ms.value / 1e9:.1f} TF/s", flush=True)
    eng.close(); del eng; torch.cuda.empty_cache()
