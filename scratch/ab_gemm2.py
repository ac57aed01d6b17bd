import torch, sys, os
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
onchip = os.environ.get("ONCHIP") == "1"
def bench(M, N, K, a_t, b_t, it=20):
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda")
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda")
    As, Bs = G.split(A), G.split(B)
    C = torch.empty(M, N, device="cuda")
    if onchip:
        f = lambda: G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N, onchip=True)
    else:
        f = lambda: G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N, a_small=As, b_small=Bs)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"M={M} N={N} K={K} a_t={a_t} b_t={b_t}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.1f} TF/s")
bench(8192, 768, 50264, False, True)
bench(8192, 3072, 768, False, False)
bench(768, 3072, 8192, True, False)
bench(1024, 64, 1024, False, False)
