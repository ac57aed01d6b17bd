"""TMEM-A GEMM path vs the shared-memory path (both on-chip residuals): bitwise, and vs float64."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
out = {}
S, dh = 1024, 64
torch.manual_seed(0)
for name, (M, N, K, Z) in {"attn": (S, dh, S, 12), "plain": (256, 64, 512, 1), "ragged": (300, 40, 200, 1)}.items():
    A = torch.rand(Z, M, K, device="cuda")
    B = torch.randn(Z, K, N, device="cuda")
    C = torch.empty(Z, M, N, device="cuda")
    G.gemm(M, N, K, A, K, False, B, N, True, C, N, z1=Z, sa=(M * K, 0), sb=(K * N, 0), sc=(M * N, 0), onchip=True)
    A2 = torch.rand(Z, M, K, device="cuda"); B2 = torch.randn(Z, K, N, device="cuda")
    D = torch.zeros(Z, M, N, device="cuda")
    G.gemm_dual(M, N, K, A, K, False, B, N, True, A2, K, B2, N, D, N, z1=Z, sa=(M * K, 0), sb=(K * N, 0),
                sa2=(M * K, 0), sb2=(K * N, 0), sc=(M * N, 0), onchip=True)
    torch.cuda.synchronize()
    ref = A.double() @ B.double()
    rel = float((C.double() - ref).norm() / ref.norm())
    ref2 = ref + A2.double() @ B2.double()
    rel2 = float((D.double() - ref2).norm() / ref2.norm())
    out[name] = (C.cpu(), D.cpu())
    print(name, "rel", rel, "dual rel", rel2, flush=True)
torch.save(out, sys.argv[1])
