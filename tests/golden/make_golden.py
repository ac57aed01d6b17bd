"""Generates tests/golden/reference_golden.npz from the COMPILED REFERENCE
(oracle/_ref/libspecden_ref.so, built from /root/reference/proj/src by
oracle/build_ref.sh). Run here, where /root/reference exists; the fixture
travels to the GPU box, the reference does not.

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import pyoracle  # noqa: E402

F32, F64 = pyoracle.F32, pyoracle.F64


def main():
    pyoracle.build()
    r = pyoracle.Reference()
    out = {}
    # probes: dims straddling the 1024 grid, both precisions, 3 distributions
    for dim in (4, 5, 129, 1025, 2050, 5000):
        for prec in (F32, F64):
            for dist, name in ((0, "gauss"), (1, "rad")):
                for seed in (42, 99):
                    out[f"probe_{name}_{dim}_{prec}_{seed}"] = r.draw_probe(dim, 3, seed, dist, prec=prec)
    out["probe_onehot_5_2"] = r.draw_probe(5, 2, 0, 2, 2, normalize=False)
    # dot / axpy / scale on counter-Gaussian inputs (f32 inputs pre-rounded)
    for dim in (1000, 1025, 5000, 70001):
        for prec in (F32, F64):
            a = pyoracle.oracle().gaussian_fill(21, 0, dim)
            b = pyoracle.oracle().gaussian_fill(22, 0, dim)
            if prec == F32:
                a = a.astype(np.float32).astype(np.float64)
                b = b.astype(np.float32).astype(np.float64)
            out[f"dot_{dim}_{prec}"] = np.array([r.dot(a, b, workers=7, prec=prec)])
            out[f"axpy_{dim}_{prec}"] = r.axpy(0.7, a, b, workers=3, prec=prec)
            out[f"scale_{dim}_{prec}"] = r.scale(a, -1.25, workers=3, prec=prec)
    # dense operators and their apply
    out["wigner_64_1_3"] = r.wigner(64, 1.0, 3)
    out["spiked_128_1_2"] = r.spiked(128, 1.0, [40.0, -35.0], 2)
    W = r.wigner(512, 1.0, 0)
    for prec in (F32, F64):
        x = r.draw_probe(512, 1, 7, 0, prec=prec)
        out[f"wigner512_apply_{prec}"] = r.dense_apply(W, x, workers=5, prec=prec)
    # Lanczos composed from the reference primitives
    S = r.spiked(256, 1.0, [50.0, -50.0], 5)
    for prec in (F32, F64):
        for reorth in (0, 1):
            for dist in (0, 1):
                res = r.lanczos_dense(S, 25, workers=4, reorth=reorth, seed=42, dist=dist, prec=prec)
                out[f"lanczos_spiked256_{prec}_{reorth}_{dist}_alpha"] = res["alphas"]
                out[f"lanczos_spiked256_{prec}_{reorth}_{dist}_beta"] = res["betas"]
    np.savez_compressed(Path(__file__).with_name("reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
