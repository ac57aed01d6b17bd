"""Epilogue cost: beta = 0 (TMA-store epilogue) vs beta = 1 (register epilogue reading C),
hot L2 vs flushed L2, for the d-wide outputs of the HVP."""
import torch, sys
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
def bench(M, N, K, b_t, beta, cold, it=30):
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda")
    As, Bs = G.split(A), G.split(B)
    C = torch.zeros(M, N, device="cuda")
    f = lambda: G.gemm(M, N, K, A, K, False, B, B.shape[1], not b_t, C, N, beta=beta, a_small=As, b_small=Bs)
    for _ in range(3): f()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(it):
        if cold: flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / it
    print(f"M={M} N={N} K={K} b_t={b_t} beta={beta} cold={cold}: {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TF/s", flush=True)
for sh in [(8192, 768, 768, False), (8192, 768, 768, True), (8192, 768, 3072, False)]:
    for beta in (0.0, 1.0):
        for cold in (False, True):
            bench(*sh, beta, cold)
