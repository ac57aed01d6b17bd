"""The NCCL plumbing on one GPU: a single-rank communicator (legal on one
device: no rank waits on another) drives the data-sharded HVP operator
(all-reduce) and the sharded Lanczos scalar exchange (all-gather + rank
fold). Results must equal the communicator-free runs bit for bit."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.distributed as dist
    import paper_2505_11564_b200 as sd
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    c = sd.nccl_comm()
    yield c
    c.close()
    dist.destroy_process_group()


def test_gpt_operator_allreduce_and_lanczos_exchange(comm):
    import paper_2505_11564_b200 as sd
    from paper_2505_11564_b200 import gpt
    cfg = dict(n_layer=2, d=64, n_head=4, ff=256, vocab=128, ctx=64)
    eng = gpt.GptHvp(cfg, 2, 64)
    lc = sd.LanczosConfig(k_max=6, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                          probe=sd.ProbeSpec(seed=3, distribution=sd.RADEMACHER))
    a = sd.lanczos_run(eng.operator(), lc)
    b = sd.lanczos_run(eng.operator(comm), lc, comm=comm)
    assert np.array_equal(a.alphas, b.alphas) and np.array_equal(a.betas, b.betas)


def test_dense_sharded_lanczos_with_comm(comm):
    import paper_2505_11564_b200 as sd
    op = sd.spiked_operator(256, 1.0, [50.0, -50.0], 5)
    lc = sd.LanczosConfig(k_max=20, reorthogonalize=sd.REORTH_FULL, prec=sd.F64,
                          probe=sd.ProbeSpec(seed=42, distribution=sd.RADEMACHER))
    a = sd.lanczos_run(op, lc)
    b = sd.lanczos_run(op, lc, comm=comm)
    assert np.array_equal(a.alphas, b.alphas) and np.array_equal(a.betas, b.betas)


def test_sharded_gpt_operator_one_rank(comm):
    # parameter-sharded Lanczos over the data-sharded HVP: all-gather x,
    # reduce-scatter Hv (NCCL, one rank) == the plain operator, bit for bit
    import paper_2505_11564_b200 as sd
    from paper_2505_11564_b200 import gpt
    cfg = dict(n_layer=1, d=64, n_head=4, ff=256, vocab=96, ctx=32)
    eng = gpt.GptHvp(cfg, 2, 32)
    lc = sd.LanczosConfig(k_max=5, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                          probe=sd.ProbeSpec(seed=9, distribution=sd.RADEMACHER))
    layout = sd.split_evenly(eng.P, 1)
    a = sd.lanczos_run(eng.operator(), lc)
    b = sd.lanczos_run(eng.operator(comm, layout=layout), lc, layout=layout, comm=comm)
    assert np.array_equal(a.alphas, b.alphas) and np.array_equal(a.betas, b.betas)


def test_operator_destroy_releases_contexts(comm):
    # the sharded operator owns three full-length scratch vectors: creating and
    # dropping it repeatedly must not grow device memory
    import gc
    import paper_2505_11564_b200 as sd
    from paper_2505_11564_b200 import gpt
    cfg = dict(n_layer=1, d=64, n_head=4, ff=256, vocab=96, ctx=32)
    eng = gpt.GptHvp(cfg, 2, 32)
    layout = sd.split_evenly(eng.P, 1)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(40):
        op = eng.operator(comm, layout=layout)
        del op
        gc.collect()
    torch.cuda.synchronize()
    assert free0 - torch.cuda.mem_get_info()[0] < 8 * eng.P * 4  # would be 40 x 3 x P floats if leaked
