"""Is the 64-wide attention product (P . v: A = P K-major [Z][1024][1024], B = v
MN-major [Z][1024][64], on-chip residuals) bound by its DRAM access pattern?
Same per-tile work with P L2-resident (Z = 18, 75 MB, hot) vs streamed from
HBM (Z = 96 / Z = 18 with an L2 flush)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2505_11564_b200 import gemm as G
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
S, dh = 1024, 64
for Z, cold in ((96, False), (18, False), (18, True), (36, False)):
    P = torch.rand(Z, S, S, device="cuda")
    V = torch.randn(Z, S, dh, device="cuda")
    O = torch.empty(Z, S, dh, device="cuda")
    f = lambda: G.gemm(S, dh, S, P, S, False, V, dh, True, O, dh, z1=Z, sa=(S * S, 0), sb=(S * dh, 0),
                       sc=(S * dh, 0), onchip=True)
    for _ in range(3): f()
    torch.cuda.synchronize()
    tot, it = 0.0, 20
    for _ in range(it):
        if cold: flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / it
    tiles = Z * S // 128
    waves = -(-tiles // 148)
    print(f"Z={Z:3d} cold={cold}: {ms*1e3:8.1f} us  {2*Z*S*S*dh/ms/1e9:6.1f} TF/s  tiles {tiles} waves {waves}  us/wave {ms*1e3/waves:.1f}", flush=True)
    del P, V, O
