"""TEST INFRASTRUCTURE: end-to-end SLQ parity on BASELINE configs[0] (C1).

C1 = SPEC's small transformer (SPEC.md:178-181 `attention_block` + cross
entropy; SURVEY Appendix C dims): one GPT block, d = 64, 4 heads, S = 32,
V = 64, batch 4, fp32; one Rademacher probe (seed 42), 32 Lanczos steps, full
reorthogonalisation. The GPU run (device HVP engine + device Lanczos engine,
both sd_* in libspecden_b200.so) is compared with the CPU run of the same
configuration (oracle: lanczos_run restatement over the oracle's Graph HVP,
oracle/src/capi.cpp oracle_lanczos_gpt), quantity by quantity:

  alpha/beta        max |d| <= 5e-5 * ||T||_max
  Ritz values        max |d| <= 2e-5 * (theta_max - theta_min)
  Ritz weights (first components^2)     max |d| <= 2e-5
  moments m <= 2k-1       |d_m|  <= 2e-5 * max(1, m) * sum_i w_i |theta_i|^m

The CPU reference is the f64 tape with f32-rounded Lanczos vectors (the
reference's f32 mode stores f32-representable values). The GPU HVP is within
~4e-6 rel-L2 of an f64 HVP (the north star's 1e-5 HVP tolerance); an HVP
perturbation of relative size e moves alpha/beta by up to ~e*||H|| and every
Ritz value by up to ~e*||H||, and the m-th moment sum w theta^m by up to
~m * e * sum w |theta|^m (the derivative of theta^m), hence the tolerances
(measured on B200: alpha 1.6e-5, moments at m = 63 2e-4 = 3.2e-6 * m). The
oracle's own f32-tape run differs from the f64-tape run by <= 1e-6.
"""
from __future__ import annotations

import numpy as np

C1 = dict(n_layer=1, d=64, n_head=4, ff=256, vocab=64, ctx=32)
B, S, K, SEED = 4, 32, 32, 42
TOL = {"alpha": 5e-5, "beta": 5e-5, "ritz_values": 2e-5, "ritz_weights": 2e-5, "moments": 2e-5}


def cpu_run(oracle):
    th = oracle.gpt_init(C1, 0, 0.0, 0.0, prec=0)
    tok, tgt = oracle.gpt_batch(C1, B, S)
    r = oracle.lanczos_gpt(C1, th, tok, tgt, B, S, K, reorth=True, seed=SEED, dist=1, prec=0, hvp_prec=1)
    v, w = oracle.ritz(r["alphas"], r["betas"])
    return r["alphas"], r["betas"], v, w, th, tok, tgt


def gpu_run(sd, gpt, th=None):
    eng = gpt.GptHvp(C1, B, S, init_seed=0)
    if th is not None:
        assert np.array_equal(eng.theta_numpy(), th), "synthetic init differs from the oracle's"
    cfg = sd.LanczosConfig(k_max=K, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                           probe=sd.ProbeSpec(seed=SEED, distribution=sd.RADEMACHER))
    res = sd.lanczos_run(eng.operator(), cfg)
    rz = sd.ritz_decompose(res.alphas, res.betas)
    eng.close()
    return res.alphas, res.betas, rz.values, rz.weights


def compare(gpu, cpu) -> dict:
    ag, bg, vg, wg = gpu
    ac, bc, vc, wc = cpu[:4]
    assert ag.size == ac.size == K and bg.size == bc.size == K - 1, (ag.size, ac.size)
    tnorm = max(np.max(np.abs(ac)), np.max(np.abs(bc)))
    err = {
        "alpha": float(np.max(np.abs(ag - ac)) / tnorm),
        "beta": float(np.max(np.abs(bg - bc)) / tnorm),
        "ritz_values": float(np.max(np.abs(vg - vc)) / (vc[-1] - vc[0])),
        "ritz_weights": float(np.max(np.abs(wg - wc))),
    }
    mom = 0.0
    for m in range(2 * K):
        mc = np.sum(wc * vc ** m)
        mg = np.sum(wg * vg ** m)
        mom = max(mom, float(abs(mg - mc) / np.sum(wc * np.abs(vc) ** m)) / max(1, m))
    err["moments"] = mom  # already divided by max(1, m)
    bad = {k: v for k, v in err.items() if not v <= TOL[k]}
    assert not bad, f"C1 SLQ parity outside {TOL}: {bad}"
    return err
