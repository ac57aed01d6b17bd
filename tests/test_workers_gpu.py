"""Multi-worker SLQ on one B200 with in-process workers (sd_comm_local_create:
the reference's WorkerPool model -- one host thread and one stream per worker,
exchanges by device copies between host barriers; no kernel waits on another
worker's kernel). This runs the multi-rank code paths of the product end to
end with real data: sharded Lanczos vectors, all-gathered f64 partials folded
in rank order, gathered operator inputs, data-sharded HVPs reduce-scattered.

SPEC acceptance 3: full SLQ pipeline with 1 vs 8 workers on an
identical config -- bitwise-identical spectrum CSVs in f64 mode; relative
Ritz-value differences < 2e-6 in f32 mode (here: bitwise as well)."""
import filecmp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sd():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2505_11564_b200 as sd
    return sd


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("reorth", ["none", "full"])
def test_acceptance3_one_vs_eight_workers(sd, tmp_path, prec, reorth):
    from paper_2505_11564_b200 import slq
    n = 256
    op = sd.wigner_operator(n, 1.0, 11)
    cfg = sd.LanczosConfig(k_max=10, prec=sd.F64 if prec == "f64" else sd.F32,
                           reorthogonalize=sd.REORTH_FULL if reorth == "full" else sd.REORTH_NONE,
                           probe=sd.ProbeSpec(seed=0, distribution=sd.GAUSSIAN))
    seeds = [0, 1, 2]
    one = tmp_path / "w1"
    a = slq.slq(op, cfg, seeds, out_dir=str(one))
    lay = sd.split_evenly(n, 8)

    def worker(r, comm):
        return slq.slq(op, cfg, seeds, out_dir=str(tmp_path / f"w8_{r}"), layout=lay, comm=comm)

    res = sd.run_workers(8, worker)
    for r in range(8):
        assert np.array_equal(res[r].spectrum.values, a.spectrum.values)
        assert np.array_equal(res[r].spectrum.weights, a.spectrum.weights)
    for f in sorted(os.listdir(one)):
        if f.endswith(".csv"):
            assert filecmp.cmp(one / f, tmp_path / "w8_0" / f, shallow=False), f


def test_dense_lanczos_workers_match_reference_fold(sd, oracle):
    # sharded Lanczos on a spiked operator, 5 workers (ragged shards) == the
    # oracle's single-worker run, bit for bit (alpha/beta)
    S = sd.spiked_dense(300, 1.0, [40.0, -40.0], 3)
    op = sd.dense_operator(S)
    cfg = sd.LanczosConfig(k_max=14, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                           probe=sd.ProbeSpec(seed=42, distribution=sd.RADEMACHER))
    ref = oracle.lanczos_dense(S, 14, reorth=True, seed=42, dist=1, prec=0)
    lay = sd.split_evenly(300, 5)
    out = sd.run_workers(5, lambda r, c: sd.lanczos_run(op, cfg, layout=lay, comm=c))
    for r in out:
        assert np.array_equal(r.alphas, ref["alphas"]) and np.array_equal(r.betas, ref["betas"])


def test_data_sharded_gpt_workers(sd):
    # two workers, each with half of the batch (loss scale 1/T_global), Lanczos
    # vectors split between them: all-gather q, reduce-scatter Hv
    # (sd_operator_gpt_sharded) -- vs one worker on the whole batch
    from paper_2505_11564_b200 import gpt
    cfg = dict(n_layer=2, d=64, n_head=4, ff=128, vocab=96, ctx=32)
    B, S = 4, 32
    tok, tgt = gpt.synthetic_tokens(cfg["vocab"], B, S, seed=1)
    lc = sd.LanczosConfig(k_max=8, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                          probe=sd.ProbeSpec(seed=5, distribution=sd.RADEMACHER))
    whole = gpt.GptHvp(cfg, B, S, init_seed=0, gain_scale=0.1, tokens=tok, targets=tgt)
    a = sd.lanczos_run(whole.operator(), lc)
    lay = sd.split_evenly(whole.P, 2)

    def worker(r, comm):
        sl = slice(r * (B // 2) * S, (r + 1) * (B // 2) * S)
        eng = gpt.GptHvp(cfg, B // 2, S, theta=whole.theta, tokens=tok[sl], targets=tgt[sl], loss_scale=1.0 / (B * S))
        return sd.lanczos_run(eng.operator(comm, layout=lay), lc, layout=lay, comm=comm)

    out = sd.run_workers(2, worker)
    assert np.array_equal(out[0].alphas, out[1].alphas) and np.array_equal(out[0].betas, out[1].betas)
    np.testing.assert_allclose(out[0].alphas, a.alphas, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(out[0].betas, a.betas, rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("n_stages,M", [(2, 3), (4, 5)])
def test_pipeline_operator_workers(sd, n_stages, M):
    # the pipeline-parallel operator end to end with in-process workers: the
    # 1F1B schedule's grouped send/recv between stage workers, Lanczos vectors
    # sharded by the stages' parameter slices -- alpha/beta bitwise equal to the
    # one-stage engine with the same micro-batches (and, with lean engine flags
    # and bf16 weights, to its own one-stage run)
    from paper_2505_11564_b200 import gpt
    for cfg, flags in ((dict(n_layer=4, d=64, n_head=4, ff=96, vocab=96, ctx=32, arch=1, rope_base=1e4), {}),
                       (dict(n_layer=4, d=64, n_head=4, ff=96, vocab=96, ctx=32, arch=1, rope_base=1e4, n_kv_head=2,
                             bf16_weights=1), dict(recompute=True, probe_residual=False))):
        S = 32
        tok, tgt = gpt.synthetic_tokens(cfg["vocab"], M, S, seed=1)
        lc = sd.LanczosConfig(k_max=6, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                              probe=sd.ProbeSpec(seed=3, distribution=sd.RADEMACHER))
        P = gpt.param_count(cfg)
        theta = gpt.init_params_range(cfg, 0, P, init_seed=0, gain_scale=0.1)
        whole = gpt.GptStage(cfg, 1, S, M, 0, cfg["n_layer"], theta, n_sets=1, tokens=tok, targets=tgt, **flags)
        lay1 = gpt.pipeline_layout(cfg, 1)
        a = sd.run_workers(1, lambda r, c: sd.lanczos_run(whole.operator(c), lc, layout=lay1, comm=c))[0]
        lay = gpt.pipeline_layout(cfg, n_stages)
        ranges = gpt.pipeline_layers(cfg["n_layer"], n_stages)

        def worker(r, comm):
            l0, l1 = ranges[r]
            b, e = lay.shard_bounds[r]
            st = gpt.GptStage(cfg, 1, S, M, l0, l1, theta[b:e], n_sets=min(M, n_stages - r), tokens=tok,
                              targets=tgt, **flags)
            return sd.lanczos_run(st.operator(comm), lc, layout=lay, comm=comm)

        out = sd.run_workers(n_stages, worker)
        for res in out:
            assert np.array_equal(res.alphas, a.alphas) and np.array_equal(res.betas, a.betas)


@pytest.mark.timeout(120)
def test_failing_worker_aborts_the_group(sd):
    # pool.cpp:54-64: every worker replies, the first (lowest-rank) exception is
    # rethrown. A worker failing outside a collective aborts the group, so the
    # others leave their waits instead of hanging; the original error surfaces.
    op = sd.wigner_operator(128, 1.0, 3)
    cfg = sd.LanczosConfig(k_max=5, prec=sd.F64, probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER))
    lay = sd.split_evenly(128, 3)

    def worker(r, comm):
        if r == 1:
            raise ValueError("worker 1 failed")
        return sd.lanczos_run(op, cfg, layout=lay, comm=comm)

    with pytest.raises(ValueError, match="worker 1 failed"):
        sd.run_workers(3, worker)
    # the device and new groups are still usable afterwards
    out = sd.run_workers(3, lambda r, c: sd.lanczos_run(op, cfg, layout=lay, comm=c))
    ref = sd.lanczos_run(op, cfg)
    assert np.array_equal(out[2].alphas, ref.alphas)
