"""TMEM-A for MN-major A (the P^T products) vs the shared-memory path: bitwise."""
import sys, torch
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
torch.manual_seed(1)
out = {}
for name, (M, N, K, Z) in {"attnT": (1024, 64, 1024, 12), "plain": (256, 64, 512, 1), "ragged": (300, 40, 200, 1)}.items():
    A = torch.rand(Z, K, M, device="cuda")  # A stored K x M (MN-major operand)
    B = torch.randn(Z, K, N, device="cuda")
    C = torch.empty(Z, M, N, device="cuda")
    G.gemm(M, N, K, A, M, True, B, N, True, C, N, z1=Z, sa=(M * K, 0), sb=(K * N, 0), sc=(M * N, 0), onchip=True)
    torch.cuda.synchronize()
    ref = A.double().transpose(1, 2) @ B.double()
    print(name, "rel", float((C.double() - ref).norm() / ref.norm()), flush=True)
    out[name] = C.cpu()
torch.save(out, sys.argv[1])
