import torch, sys
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
torch.manual_seed(0)
def rel(a,b): return float((a.double()-b).norm()/b.norm())
for K in (32, 256, 768, 3072):
    A = torch.randn(512, K, device="cuda"); B = torch.randn(K, 512, device="cuda")
    ref = A.double() @ B.double()
    f32 = rel(A @ B, ref) if True else 0
    torch.backends.cuda.matmul.allow_tf32 = False
    f32 = rel(torch.matmul(A, B), ref)
    print(K, "trunc-split", rel(G.matmul(A, B, True, mode=0), ref), "rna-split", rel(G.matmul(A, B, True, mode=1), ref), "1x", rel(G.matmul(A, B, False), ref), "torch fp32", f32)
# probe hardware conversion: a = 1 + 2^-12 (below tf32 precision), b = 1
for val in [1 + 2**-12, 1 + 3 * 2**-12, 1 + 2**-11 + 2**-12]:
    A = torch.full((128, 32), 0.0, device="cuda"); A[:, 0] = val
    B = torch.zeros(32, 128, device="cuda"); B[0, :] = 1.0
    C = G.matmul(A, B, False)
    print(f"tf32 read of {val!r}: {C[0,0].item()!r}  trunc={1+ (int((val-1)*2**10))/2**10!r}")
