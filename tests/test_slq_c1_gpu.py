"""BASELINE configs[0] (C1) end to end: device HVP + device Lanczos (fp32,
full reorth, 32 steps, one Rademacher probe) vs the CPU oracle run of the same
configuration -- alpha/beta, Ritz values, Ritz weights and the Gauss moments
m <= 2k-1, each within the tolerance stated in tests/slq_c1.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_c1_slq_parity(oracle):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2505_11564_b200 as sd
    from paper_2505_11564_b200 import gpt

    import slq_c1
    cpu = slq_c1.cpu_run(oracle)
    gpu = slq_c1.gpu_run(sd, gpt, th=cpu[4])
    err = slq_c1.compare(gpu, cpu)
    print("C1 SLQ parity:", err)
    # the spectral density built from both runs, on the
    # same grid: a Ritz shift d moves a Gaussian of width sigma by ~d/sigma of
    # its peak, so the tolerance is the Ritz tolerance x width / sigma
    sigma = 0.1
    dg = sd.smooth_density(sd.RitzSpectrum(gpu[2], gpu[3], 0.0), sigma=sigma)
    x = dg.grid
    dc = (cpu[3][None, :] * np.exp(-0.5 * ((x[:, None] - cpu[2][None, :]) / sigma) ** 2)).sum(1) / (
        sigma * np.sqrt(2 * np.pi))
    width = cpu[2][-1] - cpu[2][0]
    assert np.max(np.abs(dg.density - dc)) <= slq_c1.TOL["ritz_values"] * width / sigma * np.max(dc)
