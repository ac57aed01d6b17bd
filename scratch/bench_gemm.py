import torch, sys
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
def bench(M, N, K, a_t, b_t, three=True, it=20):
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda")
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda")
    As, Bs = G.split(A), G.split(B)
    C = torch.empty(M, N, device="cuda")
    f = lambda: G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N, a_small=As if three else None, b_small=Bs if three else None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    tf = 2 * M * N * K / ms / 1e9
    print(f"M={M} N={N} K={K} a_t={a_t} b_t={b_t} three={three}: {ms:.3f} ms  {tf:.1f} TFLOP/s (algorithmic 2MNK)")
bench(8192, 3072, 768, False, False)
bench(8192, 768, 3072, False, False)
bench(8192, 768, 3072, False, True)
bench(768, 3072, 8192, True, False)
bench(8192, 3072, 768, False, False, three=False)
torch.backends.cuda.matmul.allow_tf32 = True
A = torch.randn(8192, 768, device="cuda"); B = torch.randn(768, 3072, device="cuda")
for _ in range(3): A @ B
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
for _ in range(20): A @ B
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/20
print(f"cuBLAS TF32 8192x3072x768: {ms:.3f} ms {2*8192*3072*768/ms/1e9:.1f} TFLOP/s")
torch.backends.cuda.matmul.allow_tf32 = False
e0.record()
for _ in range(20): A @ B
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/20
print(f"cuBLAS FP32 8192x3072x768: {ms:.3f} ms {2*8192*3072*768/ms/1e9:.1f} TFLOP/s")
