"""Host logic of the pipeline-parallel HVP (CPU, no GPU): the 1F1B schedule
(sd_pipeline_schedule, the product's own C function) and the stage parameter
slices.
  * every stage runs F and B of every micro-batch once, B(m) after F(m),
    micro-batches finish in order and at most n_stages - stage are in flight
    (the activation sets a stage allocates);
  * a blocking-semantics simulation (a lone send/recv waits for its partner,
    a group completes when all its partners are posted) never deadlocks and
    pairs every message with the same micro-batch on both sides;
  * the same schedules executed by 2 and 4 gloo ranks with real
    send/recv move each stage's boundary messages to the right peer;
  * the stage slices tile the flat parameter vector exactly as a contiguous
    ShardLayout (layout.hpp:45-55) at the C4/C5 shapes."""

import pytest

from test_multirank_gloo import run_world


@pytest.fixture(scope="module")
def gpt():
    from paper_2505_11564_b200 import gpt
    return gpt


def _units(gpt, ops):
    """Split a schedule into execution units: single ops or GROUP_BEGIN..END."""
    out, i = [], 0
    while i < len(ops):
        if ops[i][0] == gpt.PIPE_GROUP_BEGIN:
            j = i + 1
            while ops[j][0] != gpt.PIPE_GROUP_END:
                j += 1
            out.append(ops[i + 1:j])
            i = j + 1
        else:
            out.append([ops[i]])
            i += 1
    return out


def _simulate(gpt, n_stages, M):
    """Blocking-semantics execution of all stages' schedules; returns the
    per-stage order of compute ops."""
    units = [_units(gpt, gpt.pipeline_schedule(n_stages, s, M)) for s in range(n_stages)]
    pc = [0] * n_stages
    peer = {gpt.PIPE_SEND_F: 1, gpt.PIPE_RECV_F: -1, gpt.PIPE_SEND_B: -1, gpt.PIPE_RECV_B: 1}
    match = {gpt.PIPE_SEND_F: gpt.PIPE_RECV_F, gpt.PIPE_RECV_F: gpt.PIPE_SEND_F,
             gpt.PIPE_SEND_B: gpt.PIPE_RECV_B, gpt.PIPE_RECV_B: gpt.PIPE_SEND_B}
    done = [[] for _ in range(n_stages)]

    def posted(s, op):  # is `op` (kind, m) in stage s's current unit?
        return pc[s] < len(units[s]) and op in units[s][pc[s]]

    sat = set()  # (stage, unit index, op): comm ops whose partner has been posted
    while any(pc[s] < len(units[s]) for s in range(n_stages)):
        moved = False
        for s in range(n_stages):
            if pc[s] >= len(units[s]):
                continue
            for k, m in units[s][pc[s]]:
                if k in peer and (s, pc[s], (k, m)) not in sat:
                    p = s + peer[k]
                    assert 0 <= p < n_stages, (s, k)
                    if posted(p, (match[k], m)):  # the pair completes on both sides
                        sat.add((s, pc[s], (k, m)))
                        sat.add((p, pc[p], (match[k], m)))
        for s in range(n_stages):
            if pc[s] >= len(units[s]):
                continue
            u = units[s][pc[s]]
            if all(k not in peer or (s, pc[s], (k, m)) in sat for k, m in u):
                done[s].extend(op for op in u if op[0] in (gpt.PIPE_F, gpt.PIPE_B))
                pc[s] += 1
                moved = True
        assert moved, f"deadlock at S={n_stages} M={M}: {pc}"
    return done


@pytest.mark.parametrize("n_stages", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("M", [1, 2, 5, 8, 16])
def test_schedule_properties(gpt, n_stages, M):
    for s in range(n_stages):
        ops = gpt.pipeline_schedule(n_stages, s, M)
        comp = [(k, m) for k, m in ops if k in (gpt.PIPE_F, gpt.PIPE_B)]
        assert sorted(m for k, m in comp if k == gpt.PIPE_F) == list(range(M))
        assert [m for k, m in comp if k == gpt.PIPE_B] == list(range(M))  # in order
        live, peak = set(), 0
        for k, m in comp:
            if k == gpt.PIPE_F:
                live.add(m)
                peak = max(peak, len(live))
            else:
                assert m in live
                live.remove(m)
        assert peak <= min(M, n_stages - s)
        # message counts: one per micro-batch per boundary and direction
        cnt = {k: sum(1 for kk, _ in ops if kk == k) for k in range(8)}
        assert cnt[gpt.PIPE_SEND_F] == cnt[gpt.PIPE_RECV_B] == (M if s < n_stages - 1 else 0)
        assert cnt[gpt.PIPE_RECV_F] == cnt[gpt.PIPE_SEND_B] == (M if s > 0 else 0)
        assert cnt[gpt.PIPE_GROUP_BEGIN] == cnt[gpt.PIPE_GROUP_END]


@pytest.mark.parametrize("n_stages", [2, 3, 4, 8])
@pytest.mark.parametrize("M", [1, 3, 8, 13])
def test_schedule_deadlock_free(gpt, n_stages, M):
    _simulate(gpt, n_stages, M)


def test_schedule_errors(gpt):
    import paper_2505_11564_b200 as sd
    for a in ((0, 0, 1), (2, 2, 1), (2, -1, 1), (2, 0, 0)):
        with pytest.raises(sd.ArgumentError):
            gpt.pipeline_schedule(*a)


def test_stage_slices_tile_the_layout(gpt):
    import paper_2505_11564_b200 as sd
    for cfg in (gpt.LLAMA2_7B, gpt.LLAMA_70B, dict(n_layer=5, d=64, n_head=4, ff=96, vocab=96, ctx=32, arch=1,
                                                      rope_base=1e4, n_kv_head=2)):
        P = gpt.param_count(cfg)
        slots = gpt.param_layout(cfg)
        for n in (1, 2, 3, 4, 8):
            if n > cfg["n_layer"]:
                continue
            lay = gpt.pipeline_layout(cfg, n)
            sd.validate_layout(lay)
            assert lay.total_dim == P and lay.begins[0] == 0 and lay.ends[-1] == P
            starts = {o for o, _, _, _ in slots}
            assert all(b in starts for b in lay.begins)  # stage boundaries fall on parameter slots
            rng = gpt.pipeline_layers(cfg["n_layer"], n)
            assert rng[0][0] == 0 and rng[-1][1] == cfg["n_layer"]
            assert all(rng[i][1] == rng[i + 1][0] for i in range(n - 1))
            # the embedding sits on stage 0, the head on the last stage
            assert lay.ends[0] > slots[0][0] + slots[0][1] * slots[0][2] - 1
            assert lay.begins[-1] <= slots[-1][0]


def _gloo_pipeline(rank, world):
    """Each rank = one stage running its schedule with gloo send/recv; a
    stage's forward output for micro-batch m is (m, stage) tagged data, its
    backward output likewise; receivers check what arrives."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist
    from paper_2505_11564_b200 import gpt
    M, n = 5, 16
    ops = gpt.pipeline_schedule(world, rank, M)
    xbuf, gbuf = {}, {}
    log = []
    pending = []

    def fwd_payload(s, m):
        return torch.arange(n, dtype=torch.float32) + 1000.0 * m + 100.0 * s

    def bwd_payload(s, m):
        return -(torch.arange(n, dtype=torch.float32) + 1000.0 * m + 100.0 * s)

    in_group = False
    for k, m in ops:
        if k == gpt.PIPE_GROUP_BEGIN:
            in_group = True
            continue
        if k == gpt.PIPE_GROUP_END:
            for w in pending:
                w.wait()
            pending.clear()
            in_group = False
            continue
        if k == gpt.PIPE_F:
            if rank > 0:
                assert torch.equal(xbuf.pop(m), fwd_payload(rank - 1, m))
            log.append(("F", m))
        elif k == gpt.PIPE_B:
            if rank < world - 1:
                assert torch.equal(gbuf.pop(m), bwd_payload(rank + 1, m))
            log.append(("B", m))
        else:
            if k == gpt.PIPE_SEND_F:
                w = dist.isend(fwd_payload(rank, m), rank + 1)
            elif k == gpt.PIPE_SEND_B:
                w = dist.isend(bwd_payload(rank, m), rank - 1)
            elif k == gpt.PIPE_RECV_F:
                xbuf[m] = torch.empty(n)
                w = dist.irecv(xbuf[m], rank - 1)
            else:
                gbuf[m] = torch.empty(n)
                w = dist.irecv(gbuf[m], rank + 1)
            if in_group:
                pending.append(w)
            else:
                w.wait()
    assert not xbuf and not gbuf
    return log


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_pipeline_exchange(world):
    out = run_world(_gloo_pipeline, world=world)
    for r in range(world):
        log = out[r]
        assert isinstance(log, list), log
        assert [m for k, m in log if k == "B"] == list(range(5))
