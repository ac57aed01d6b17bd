import torch, sys
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
torch.manual_seed(0)
for (a_t, b_t) in [(False, True), (False, False), (True, True), (True, False)]:
    M = N = 128; K = 32
    A = torch.ones(*((K, M) if a_t else (M, K)), device="cuda")
    B = torch.ones(*((N, K) if b_t else (K, N)), device="cuda")
    C = torch.full((M, N), -7.0, device="cuda")
    G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N)
    torch.cuda.synchronize()
    print(a_t, b_t, "ones:", C[0, :4].tolist(), C[127, 124:].tolist(), float(C.mean()))
    A = torch.randn(*((K, M) if a_t else (M, K)), device="cuda")
    B = torch.randn(*((N, K) if b_t else (K, N)), device="cuda")
    ref = (A.t() if a_t else A) @ (B.t() if b_t else B)
    G.gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C, N)
    torch.cuda.synchronize()
    print("  randn max err", float((C - ref).abs().max()), "ref", ref[0, :3].tolist(), "got", C[0, :3].tolist())
