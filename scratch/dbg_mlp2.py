import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2505_11564_b200 import mlp
from oracle.pyoracle import Oracle
o = Oracle()
for widths, n in [([16, 32, 4], 64), ([16, 32, 4], 10), ([4, 8, 4], 64), ([16, 8, 4], 10), ([4, 32, 4], 10), ([16, 4], 10), ([4, 4], 10), ([8, 4], 10)]:
    rng = np.random.default_rng(1)
    P = mlp.param_count(widths)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    th = f32(rng.standard_normal(P) * 0.5); X = f32(rng.standard_normal((n, widths[0]))); Y = f32(rng.standard_normal((n, widths[-1])))
    eng = mlp.MlpHvp(widths, torch.tensor(th, dtype=torch.float32, device="cuda"), n_max=n, x=X, y=Y)
    v = f32(rng.standard_normal(P))
    got = eng.hvp(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    want = o.mlp_hvp(widths, th, X, Y, v)
    # numpy forward loss
    h = X; off = 0
    for l in range(len(widths) - 1):
        W = th[off:off + widths[l] * widths[l + 1]].reshape(widths[l], widths[l + 1]); off += W.size
        b = th[off:off + widths[l + 1]]; off += b.size
        h = h @ W + b
        if l + 2 < len(widths): h = np.tanh(h)
    loss = np.mean((h - Y) ** 2)
    print(widths, n, "hvp rel", np.linalg.norm(got - want) / np.linalg.norm(want), "loss", eng.loss(), loss)
