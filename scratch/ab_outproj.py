"""A/B of the tile choices for the attention out-projection shapes (8192 x 768 x 768)."""
import os, subprocess, sys
code = r'''
import torch, sys
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
def bench(M, N, K, a_t, b_t, it=50):
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda")
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda")
    As, Bs = G.split(A), G.split(B)
    C = torch.empty(M, N, device="cuda")
    f = lambda: G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N, a_small=As, b_small=Bs)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"  M={M} N={N} K={K} a_t={a_t} b_t={b_t}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.1f} TF/s")
for sh in [(8192, 768, 768, False, False), (8192, 768, 768, False, True), (768, 768, 8192, True, True),
           (8192, 768, 3072, False, False), (8192, 768, 2304, False, False), (8192, 2304, 768, False, True)]:
    bench(*sh)
'''
for env in [{}, {"SD_GEMM_PAIR": "0"}, {"SD_GEMM_PAIR_N": "192"}, {"SD_GEMM_PAIR": "0", "SD_GEMM_WIDE": "0"}]:
    print(env, flush=True)
    subprocess.run([sys.executable, "-c", code], env={**os.environ, **env})
