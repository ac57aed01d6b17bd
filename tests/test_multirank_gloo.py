"""World-size-2 gloo tests (CPU) of the multi-rank host logic that the NCCL
path runs on B200s: (1) parameter-sharded blocked partials all-gathered and
folded in rank order by the product's combine (sd_combine_partials_host) are
bitwise equal to the single-rank fold on every rank (reduction.hpp:76-107);
(2) data-sharded HVP summed by all-reduce with per-rank weight |B_r|/N equals
the whole-batch HVP (Alg. 1 lines 13-17)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surfaced to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return out


def _sharded_dot(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle.pyoracle import Oracle
    from paper_2505_11564_b200 import _lib, core
    o = Oracle()
    P = 70001
    a = o.gaussian_fill(3, 0, P)
    b = o.gaussian_fill(4, 0, P)
    lay = core.split_evenly(P, world)
    s, e = lay.shard_bounds[rank]
    head, sums, tail = o.dot_partial(s, e, P, a[s:e], b[s:e])   # this rank's partial (host restatement)
    mine = torch.tensor(np.concatenate([head, sums, tail]), dtype=torch.float64)
    pmax = max(_lib.lib().sd_partial_len(bb, ee, P) for bb, ee in lay.shard_bounds)
    buf = torch.zeros(pmax, dtype=torch.float64)
    buf[:mine.numel()] = mine
    gathered = [torch.zeros(pmax, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, buf)
    arrs = [g.numpy().copy() for g in gathered]
    ptrs = (_lib.dp * world)(*[x.ctypes.data_as(_lib.dp) for x in arrs])
    out = C.c_double()
    bb = (C.c_uint64 * world)(*lay.begins)
    ee = (C.c_uint64 * world)(*lay.ends)
    _lib.check(_lib.lib().sd_combine_partials_host(world, bb, ee, P, ptrs, C.byref(out)))
    return {"combined": out.value, "reference": o.dot(a, b)}


def test_parameter_sharded_dot_is_bitwise_rank_invariant():
    res = run_world(_sharded_dot)
    assert all(isinstance(v, dict) for v in res.values()), res
    vals = {np.float64(v["combined"]).view(np.int64) for v in res.values()}
    assert len(vals) == 1
    ref = res[0]["reference"]
    assert np.float64(res[0]["combined"]).view(np.int64) == np.float64(ref).view(np.int64)


CFG = dict(n_layer=1, d=16, n_head=2, ff=32, vocab=24, ctx=8)


def _data_sharded_hvp(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle.pyoracle import Oracle, RADEMACHER
    from paper_2505_11564_b200.gpt import synthetic_tokens
    o = Oracle()
    B, S = 4, 8
    th = o.gpt_init(CFG, 0, 0.1, 0.1)
    v = o.draw_probe(th.size, 3, RADEMACHER)
    tok, tgt = synthetic_tokens(CFG["vocab"], B, S, 1, 0)
    bl = B // world
    sl = slice(rank * bl * S, (rank + 1) * bl * S)
    u = o.gpt_hvp(CFG, th, tok[sl].astype(np.uint32), tgt[sl].astype(np.uint32), bl, S, v)
    h = torch.tensor(u * (bl / B))            # this rank's |B_r|/N share (engine: loss_scale = 1/T_global)
    dist.all_reduce(h)                        # the NCCL all-reduce of Hv on B200
    whole = o.gpt_hvp(CFG, th, tok.astype(np.uint32), tgt.astype(np.uint32), B, S, v)
    return {"rel": float(np.linalg.norm(h.numpy() - whole) / np.linalg.norm(whole))}


def test_data_sharded_hvp_allreduce_weighting():
    res = run_world(_data_sharded_hvp)
    for r in res.values():
        assert isinstance(r, dict), r
        assert r["rel"] < 1e-12


def _sharded_apply(rank, world):
    # the index math of gpt_shard_apply (csrc/sd_gpt.cu) on CPU: all-gather the
    # x shards into maxlen slots, compact, run this rank's batch HVP on the
    # full vector, lay Hv out in rank-major maxlen slots, reduce-scatter
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle.pyoracle import Oracle, RADEMACHER
    from paper_2505_11564_b200 import core
    from paper_2505_11564_b200.gpt import synthetic_tokens
    o = Oracle()
    B, S = 4, 8
    th = o.gpt_init(CFG, 0, 0.1, 0.1)
    P = th.size
    v = o.draw_probe(P, 5, RADEMACHER)
    tok, tgt = synthetic_tokens(CFG["vocab"], B, S, 1, 0)
    lay = core.split_evenly(P, world)
    b0, e0 = lay.shard_bounds[rank]
    ml = max(e - b for b, e in lay.shard_bounds)
    slot = torch.zeros(ml, dtype=torch.float64)
    slot[:e0 - b0] = torch.tensor(v[b0:e0])
    slots = [torch.zeros(ml, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(slots, slot)
    full = np.concatenate([slots[r].numpy()[:e - b] for r, (b, e) in enumerate(lay.shard_bounds)])
    bl = B // world
    sl = slice(rank * bl * S, (rank + 1) * bl * S)
    hv = o.gpt_hvp(CFG, th, tok[sl].astype(np.uint32), tgt[sl].astype(np.uint32), bl, S, full) * (bl / B)
    send = torch.zeros(world * ml, dtype=torch.float64)
    for r, (b, e) in enumerate(lay.shard_bounds):
        send[r * ml:r * ml + (e - b)] = torch.tensor(hv[b:e])
    mine = torch.zeros(ml, dtype=torch.float64)
    dist.reduce_scatter_tensor(mine, send)
    whole = o.gpt_hvp(CFG, th, tok.astype(np.uint32), tgt.astype(np.uint32), B, S, v)
    ref = whole[b0:e0]
    return {"rel": float(np.linalg.norm(mine.numpy()[:e0 - b0] - ref) / np.linalg.norm(ref)),
            "gathered_exact": bool(np.array_equal(full, v))}


def test_parameter_sharded_lanczos_apply():
    res = run_world(_sharded_apply)
    for r in res.values():
        assert isinstance(r, dict), r
        assert r["gathered_exact"] and r["rel"] < 1e-12


def test_bench_probe_partition_covers_every_probe_once():
    # bench.py --gpus N (C1/C2): rank r runs probe chains r, r + N, ... -- the
    # ranks together run the SLQ job's probes 0..n-1 exactly once, and the
    # data-sharded partition drives the same chain on every rank
    import bench
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            first, stride = bench.probe_seed_plan(0, r, world, True)
            seen += [first + i * stride for i in range(10 // world + 1) if first + i * stride < 10]
        assert sorted(seen) == list(range(10))
        assert all(bench.probe_seed_plan(42, r, world, False) == (42, 1) for r in range(world))
