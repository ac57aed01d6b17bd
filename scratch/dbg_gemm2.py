import torch, sys, ctypes as C, numpy as np
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
from paper_2505_11564_b200._lib import lib
L = lib()
dbg = torch.zeros(64 * 1024 // 4, device="cuda")
C.c_void_p.in_dll(L, "sd_gemm_debug_buffer").value = dbg.data_ptr()
M = N = 128; K = 32
# A MN-major: stored K x M, A[k][m] = m + 1000*k ; B K-major: stored N x K ones
A = (torch.arange(M, device="cuda").float()[None, :] + 1000 * torch.arange(K, device="cuda").float()[:, None]).contiguous()
B = torch.ones(N, K, device="cuda")
Cm = torch.full((M, N), -7.0, device="cuda")
G.gemm(M, N, K, A, M, True, B, K, False, Cm, N)
torch.cuda.synchronize()
d = dbg.cpu().numpy()
print("C[0,:3]", Cm[0, :3].tolist(), "C[5,:3]", Cm[5, :3].tolist(), "expect row m:", [32 * 5 + 1000 * 496])
print("A tile first 40 floats:", d[:40].tolist())
print("A tile at 1024B (k-row 8):", d[256:264].tolist())
print("A tile at 4096B (chunk 1):", d[1024:1032].tolist())
print("B tile:", d[4096:4100].tolist(), "nonzero count in A tile:", int((d[:4096] != 0).sum()))
