"""64-wide attention product: on-chip residuals vs residual arrays vs 1xTF32 (hot L2, Z = 36)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
S, dh = 1024, 64
for Z in (36, 96):
    P = torch.rand(Z, S, S, device="cuda")
    V = torch.randn(Z, S, dh, device="cuda")
    Ps, Vs = G.split(P), G.split(V)
    O = torch.empty(Z, S, dh, device="cuda")
    kw = dict(z1=Z, sa=(S * S, 0), sb=(S * dh, 0), sc=(S * dh, 0))
    for name, f in (("onchip", lambda: G.gemm(S, dh, S, P, S, False, V, dh, True, O, dh, onchip=True, **kw)),
                    ("arrays", lambda: G.gemm(S, dh, S, P, S, False, V, dh, True, O, dh, a_small=Ps, b_small=Vs, **kw)),
                    ("1xtf32", lambda: G.gemm(S, dh, S, P, S, False, V, dh, True, O, dh, **kw))):
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"Z={Z} {name}: {ms*1e3:8.1f} us  {2*Z*S*S*dh/ms/1e9:6.1f} TF/s", flush=True)
    del P, V, Ps, Vs, O
