"""Pipeline-parallel HVP (Llama-style family, BASELINE C4/C5 parameter-sharded
configs) on one GPU. The stages of an n-stage pipeline run in ONE process,
interleaved exactly as their 1F1B schedules (sd_pipeline_schedule) order them,
with device copies standing in for the NCCL boundary messages -- no rank ever
waits on another. Checks:
  * pipeline (S stages, M micro-batches) == the one-stage engine with the same
    M micro-batches, bit for bit (identical kernel sequence per micro-batch);
  * M = 1: == the monolithic engine bit for bit;
  * M > 1: == the monolithic engine over the concatenated batch to 1e-6
    (Alg. 1 batch weighting; only the Hv accumulation order differs) and the
    f64 oracle to the HVP tolerance 1e-5;
  * the NCCL pipeline operator on a one-rank communicator drives Lanczos."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5
LT = dict(n_layer=4, d=64, n_head=4, ff=96, vocab=96, ctx=32, arch=1, rope_base=10000)


@pytest.fixture(scope="module")
def gpt():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2505_11564_b200 import gpt
    return gpt


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run_pipeline(gpt, cfg, B, S, M, n_stages, theta, v, tokens, targets, n_sets=None, **flags):
    """All stages in one process in 1F1B order; returns the full Hv (concatenated stage slices)."""
    ranges = gpt.pipeline_layers(cfg["n_layer"], n_stages)
    stages, hv = [], torch.zeros_like(v)
    for s, (a, b) in enumerate(ranges):
        pb, pe = gpt.stage_params(cfg, a, b)
        ns = min(M, n_stages - s) if n_sets is None else n_sets
        st = gpt.GptStage(cfg, B, S, M, a, b, theta[pb:pe], n_sets=ns, tokens=tokens, targets=targets, **flags)
        st.begin_pass(v[pb:pe], hv[pb:pe])
        stages.append(st)
    Td = B * S * cfg["d"]
    sched = [gpt.pipeline_schedule(n_stages, s, M) for s in range(n_stages)]
    pc = [0] * n_stages
    box = {}  # (dst stage, kind, m) -> (a, b) tensors: the boundary messages
    while any(pc[s] < len(sched[s]) for s in range(n_stages)):
        progressed = False
        for s in range(n_stages):
            while pc[s] < len(sched[s]):
                k, m = sched[s][pc[s]]
                if k == gpt.PIPE_F:
                    if s > 0:
                        if (s, "F", m) not in box:
                            break
                        xi, dxi = box.pop((s, "F", m))
                    else:
                        xi = dxi = None
                    xo = dxo = None
                    if s < n_stages - 1:
                        xo, dxo = (torch.empty(Td, device="cuda") for _ in range(2))
                        box[(s + 1, "F", m)] = (xo, dxo)
                    stages[s].forward(m, xi, dxi, xo, dxo)
                elif k == gpt.PIPE_B:
                    if s < n_stages - 1:
                        if (s, "B", m) not in box:
                            break
                        gi, gdi = box.pop((s, "B", m))
                    else:
                        gi = gdi = None
                    go = gdo = None
                    if s > 0:
                        go, gdo = (torch.empty(Td, device="cuda") for _ in range(2))
                        box[(s - 1, "B", m)] = (go, gdo)
                    stages[s].backward(m, gi, gdi, go, gdo)
                pc[s] += 1
                progressed = True
        assert progressed, "pipeline schedule deadlocked"
    torch.cuda.synchronize()
    return hv, stages


def _setup(gpt, cfg, B, S, M, seed=3):
    P = gpt.param_count(cfg)
    eng = gpt.GptHvp(cfg, B * M, S, init_seed=0, gain_scale=0.1)
    g = torch.Generator(device="cuda").manual_seed(seed)
    v = torch.randn(P, device="cuda", generator=g)
    tok, tgt = gpt.synthetic_tokens(cfg["vocab"], B * M, S)
    return eng, v, tok, tgt


@pytest.mark.parametrize("cfg,n_stages", [(LT, 2), (LT, 4), (dict(LT, n_layer=3, n_kv_head=2), 3)])
def test_pipeline_one_microbatch_bitwise(gpt, cfg, n_stages):
    B, S = 2, 32
    eng, v, tok, tgt = _setup(gpt, cfg, B, S, 1)
    mono = eng.hvp(v)
    hv, _ = run_pipeline(gpt, cfg, B, S, 1, n_stages, eng.theta, v, tok, tgt)
    assert torch.equal(hv, mono)


@pytest.mark.parametrize("n_stages,M", [(2, 3), (4, 6), (3, 2)])
def test_pipeline_microbatches(gpt, oracle, n_stages, M):
    cfg, B, S = (dict(LT, n_kv_head=2) if n_stages == 3 else LT), 1, 32
    eng, v, tok, tgt = _setup(gpt, cfg, B, S, M, seed=n_stages)
    hv, stages = run_pipeline(gpt, cfg, B, S, M, n_stages, eng.theta, v, tok, tgt)
    # the one-stage engine with the same micro-batches: identical kernels per micro-batch
    whole = gpt.GptStage(cfg, B, S, M, 0, cfg["n_layer"], eng.theta, n_sets=1, tokens=tok, targets=tgt)
    hv1 = torch.zeros_like(v)
    whole.begin_pass(v, hv1)
    for m in range(M):
        whole.forward(m)
        whole.backward(m)
    torch.cuda.synchronize()
    assert torch.equal(hv, hv1)
    # the monolithic engine over the concatenated batch (Alg. 1 weighting)
    mono = eng.hvp(v)
    assert rel(hv.cpu(), mono.cpu()) < 1e-6
    assert abs(stages[-1].loss() - eng.loss()) < 1e-6
    # the f64 oracle
    th = eng.theta_numpy()
    vt, ot = v.double().cpu().numpy(), None
    ot = oracle.gpt_hvp(cfg, th, tok.astype(np.uint32), tgt.astype(np.uint32), B * M, S, vt)
    assert rel(hv.double().cpu().numpy(), ot) < TOL


def test_stage_errors(gpt):
    import paper_2505_11564_b200 as sd
    cfg = LT
    P = gpt.param_count(cfg)
    th = torch.zeros(P, device="cuda")
    with pytest.raises(sd.LayoutError):
        gpt.stage_params(cfg, 2, 2)
    with pytest.raises(sd.ArgumentError):  # more sets than micro-batches
        gpt.GptStage(cfg, 1, 32, 2, 0, 2, th[:gpt.stage_params(cfg, 0, 2)[1]], n_sets=3)
    with pytest.raises(sd.ConfigError):  # tied GPT-2 layout has no pipeline split
        gpt.stage_params(dict(LT, arch=0), 0, 2)
    b, e = gpt.stage_params(cfg, 1, 3)
    st = gpt.GptStage(cfg, 1, 32, 1, 1, 3, th[b:e])
    with pytest.raises(sd.StateError):  # no begin_pass
        st.forward(0, torch.zeros(32 * 64, device="cuda"), torch.zeros(32 * 64, device="cuda"))
    st.begin_pass(th[b:e], torch.empty(e - b, device="cuda"))
    with pytest.raises(sd.ArgumentError):  # a middle stage needs its input
        st.forward(0)
    with pytest.raises(sd.ArgumentError):
        st.forward(1, torch.zeros(32 * 64, device="cuda"), torch.zeros(32 * 64, device="cuda"))
    with pytest.raises(sd.StateError):  # loss lives on the last stage
        st.loss()


def test_pipeline_operator_one_rank_lanczos(gpt):
    # the NCCL pipeline operator on a one-rank communicator (one stage, four
    # micro-batches through ONE activation set) == the monolithic operator
    import torch.distributed as dist
    import paper_2505_11564_b200 as sd
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29537")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    comm = sd.nccl_comm()
    try:
        cfg, B, S, M = dict(LT, n_kv_head=2), 1, 32, 4
        eng, v, tok, tgt = _setup(gpt, cfg, B, S, M)
        st = gpt.GptStage(cfg, B, S, M, 0, cfg["n_layer"], eng.theta, n_sets=1, tokens=tok, targets=tgt)
        layout = gpt.pipeline_layout(cfg, 1)
        lc = sd.LanczosConfig(k_max=6, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,
                              probe=sd.ProbeSpec(seed=5, distribution=sd.RADEMACHER))
        a = sd.lanczos_run(eng.operator(), lc)
        b = sd.lanczos_run(st.operator(comm), lc, layout=layout, comm=comm)
        np.testing.assert_allclose(b.alphas, a.alphas, rtol=1e-5, atol=1e-9)
        np.testing.assert_allclose(b.betas, a.betas, rtol=1e-5, atol=1e-9)
    finally:
        comm.close()
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("bf16", [0, 1])
def test_lean_modes_bitwise(gpt, bf16):
    # the memory modes that fit BASELINE C5 per GPU: layer recomputation in the
    # backward and on-chip probe residuals (and bf16-valued weights) change no bit of Hv
    cfg, B, S, M, n_st = dict(LT, n_kv_head=2, bf16_weights=bf16), 1, 32, 3, 2
    eng, v, tok, tgt = _setup(gpt, cfg, B, S, M, seed=7)
    base, _ = run_pipeline(gpt, cfg, B, S, M, n_st, eng.theta, v, tok, tgt)
    for rc, pr in ((True, True), (False, False), (True, False)):
        hv, st = run_pipeline(gpt, cfg, B, S, M, n_st, eng.theta, v, tok, tgt, recompute=rc, probe_residual=pr)
        assert torch.equal(hv, base), (rc, pr)
    lean = gpt.stage_workspace_bytes(cfg, B, S, M, 0, 2, 2, gpt.RECOMPUTE | gpt.NO_PROBE_RESIDUAL)
    assert lean < gpt.stage_workspace_bytes(cfg, B, S, M, 0, 2, 2, 0)


def test_init_params_range_matches_full_init(gpt):
    # a stage initialises only its slice: bit-identical to that slice of the full init
    for cfg in (dict(LT, n_kv_head=2), dict(LT, bf16_weights=1)):
        full = gpt.GptHvp(cfg, 1, 32, init_seed=5, gain_scale=0.1).theta
        for a, b in gpt.pipeline_layers(cfg["n_layer"], 3):
            pb, pe = gpt.stage_params(cfg, a, b)
            assert torch.equal(gpt.init_params_range(cfg, pb, pe, init_seed=5, gain_scale=0.1), full[pb:pe])
        assert torch.equal(gpt.init_params_range(cfg, 7, 1000, init_seed=5, gain_scale=0.1), full[7:1000])
