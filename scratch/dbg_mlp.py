import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2505_11564_b200 import mlp
from oracle.pyoracle import Oracle
o = Oracle()
for widths, n in [([64, 256, 128, 10], 200), ([64, 256, 10], 200), ([64, 128, 10], 50)]:
    rng = np.random.default_rng(1)
    P = mlp.param_count(widths)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    th = f32(rng.standard_normal(P) * 0.5); X = f32(rng.standard_normal((n, widths[0]))); Y = f32(rng.standard_normal((n, widths[-1])))
    eng = mlp.MlpHvp(widths, torch.tensor(th, dtype=torch.float32, device="cuda"), n_max=n, x=X, y=Y)
    v = f32(rng.standard_normal(P))
    got = eng.hvp(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    want = o.mlp_hvp(widths, th, X, Y, v); w32 = o.mlp_hvp(widths, th, X, Y, v, prec=0)
    off = 0
    print(widths, "total", np.linalg.norm(got - want) / np.linalg.norm(want))
    for l in range(len(widths) - 1):
        for nm, sz in (("W", widths[l] * widths[l + 1]), ("b", widths[l + 1])):
            g, w = got[off:off + sz], want[off:off + sz]
            print(f"  {nm}{l}: rel {np.linalg.norm(g - w) / (np.linalg.norm(w) + 1e-30):.3e}  oracle-f32 {np.linalg.norm(w32[off:off+sz] - w) / (np.linalg.norm(w) + 1e-30):.3e}")
            off += sz
