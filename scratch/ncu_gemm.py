import torch, sys
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
M, N, K = 8192, 3072, 768
A = torch.randn(M, K, device="cuda"); B = torch.randn(K, N, device="cuda")
As, Bs = G.split(A), G.split(B)
C = torch.empty(M, N, device="cuda")
for _ in range(4):
    G.gemm(M, N, K, A, K, False, B, N, True, C, N, a_small=As, b_small=Bs)
torch.cuda.synchronize()
print("ok")
