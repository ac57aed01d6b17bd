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
    # the spectral density built from both runs agrees too
    dg = sd.smooth_density(sd.RitzSpectrum(gpu[2], gpu[3], 0.0), sigma=0.1)
    g, dc, _ = oracle.smooth_density(cpu[2], cpu[3], sigma=0.1, npts=dg.grid.size)
    assert np.max(np.abs(dg.density - dc)) <= 1e-5 * np.max(dc)
