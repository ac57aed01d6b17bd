import torch, sys
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
def run(M, N, K, onchip, it=20):
    A = torch.randn(K, M, device="cuda"); B = torch.randn(K, N, device="cuda")
    A2 = torch.randn(K, M, device="cuda"); B2 = torch.randn(K, N, device="cuda")
    As, Bs, A2s, B2s = G.split(A), G.split(B), G.split(A2), G.split(B2)
    C = torch.empty(M, N, device="cuda")
    f = lambda: G.gemm_dual(M, N, K, A, M, True, B, N, True, A2, M, B2, N, C, N, a_small=As, b_small=Bs,
                            a2_small=A2s, b2_small=B2s, onchip=onchip)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"M={M} N={N} K={K} dual onchip={onchip}: {ms:.3f} ms {4*M*N*K/ms/1e9:.1f} TF/s")
for shape in [(3072, 768, 8192), (768, 3072, 8192), (768, 2304, 8192), (50264, 768, 8192), (768, 768, 8192)]:
    for oc in (False, True):
        run(*shape, oc)
