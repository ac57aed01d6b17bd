#!/usr/bin/env python
"""Lanczos steps/s of the HessFormer SLQ hot path on B200 (BASELINE.json metric).

One step = one Lanczos iteration of PAPER.md Alg. 2 driven by the GPT HVP of
Alg. 1: a Hessian-vector product over the batch (B x S synthetic tokens) plus
the three-term recurrence plus full reorthogonalisation (2x classical
Gram-Schmidt over every stored column). Workload = BASELINE configs[1]:
GPT-2-small shape (124,439,808 params) random init, synthetic tokens, batch
8 x 1024, 10 probes x 100 Lanczos steps, full reorth, fp32 (3xTF32 GEMMs).
Timed: K steps of the probe chain centred on column k_max/2 (probes restart
every k_max steps), after W warm-up steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c1|c2|c4|c5] [--reduction tree|ordered]

N > 1 (torchrun, one rank per GPU): strong scaling of the same global batch,
data-sharded HVP (each rank B/N sequences); the Lanczos vectors are
parameter-sharded by split_evenly(P, N): each apply all-gathers q and
reduce-scatters Hv into the owners' shards, and every scalar set is one
all-gather of f64 partials folded in rank order.

The headline timed loop runs with no instrumentation; the GEMM share and
TF/s come from a separate profiled pass of a few more steps.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

MEASURED_PEAKS = ROOT / "MEASURED_PEAKS.json"
# measured per-launch DRAM bytes of the GEMMs (tools/gemm_traffic.py: ncu over every GEMM launch of one
# HVP at the bench shape) next to their algorithmic bytes
TRAFFIC_FILE = ROOT / "profiles" / "r02_gemm_traffic.json"
METRIC = "Lanczos steps/sec (HVP+reorth) at 1/2/4/8 B200; HVP/Lanczos roofline fraction"

# model dims of the workloads (plain dicts: the reference arm must not import the product package)
GPT2_SMALL = dict(n_layer=12, d=768, n_head=12, ff=3072, vocab=50257, ctx=1024)
C1_MODEL = dict(n_layer=1, d=64, n_head=4, ff=256, vocab=64, ctx=32)
# BASELINE configs[2] (C3): SURVEY 8 proposal -- 1.3B GPT-2-architecture decoder (24L, d2048, ff8192, V50257,
# ctx2048, tied head), 32 x 2048 = 65,536 tokens per HVP, data-sharded over the ranks in micro-batches of
# 1 x 2048 (optionally with recomputation); Lanczos vectors parameter-sharded, selective reorth over the 16
# newest columns (full reorth with the sharded basis from N >= 4)
C3_MODEL = dict(n_layer=24, d=2048, n_head=16, ff=8192, vocab=50257, ctx=2048)


def workload_config(args):
    """The config dict both arms print (identical by construction)."""
    if args.workload == "c1":
        return {"workload": "BASELINE configs[0] (C1): SPEC small transformer (1 block, d64, 4 heads, V64), "
                            "batch 4x32 tokens, 1 Rademacher probe x 32 Lanczos steps, full reorth, fp32",
                "model": "c1-small-transformer", "global_batch": 4, "seq_len": 32, "k_max": 32,
                "reorth": "full", "probes": 1}
    if args.workload == "c3":
        return {"workload": "BASELINE configs[2] (C3): 1.3B GPT-2-architecture decoder (24L d2048 ff8192 V50257), "
                            "32x2048 tokens per HVP data-sharded in 1x2048 micro-batches, "
                            f"k_max={args.k_max}, {args.c3_reorth} reorth",
                "model": "c3-1.3b", "params": 1315723264, "global_batch": 32, "seq_len": 2048,
                "micro_batch": 1, "k_max": args.k_max, "reorth": args.c3_reorth, "probes": 1}
    return {"workload": "BASELINE configs[1]: GPT-2-small shape 124M, batch 8x1024 tokens, "
                        "Rademacher probes, k_max=100, full reorth",
            "model": "gpt2-small", "params": 124439808, "global_batch": args.batch, "seq_len": args.seq,
            "k_max": args.k_max, "reorth": "full", "probes": 10}


def probe_seed_plan(base: int, rank: int, world: int, probes: bool):
    """(first probe seed, stride) of a rank's chains: with probe partitioning
    rank r runs seeds base + r, base + r + N, ... -- together the ranks cover
    base, base + 1, ... exactly once (the SLQ job's probes); otherwise every
    rank drives the same sharded chains base, base + 1, ..."""
    return (base + rank, world) if probes else (base, 1)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def peaks():
    try:
        d = json.loads(MEASURED_PEAKS.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback"


TF32_PEAK = ROOT / "profiles" / "tf32_peak.json"


def tf32_peak(bf16_sustained: float):
    """Dense TF32 tensor roofline: the driver-measured bf16 sustained rate of
    MEASURED_PEAKS.json / 2 (tcgen05 kind::tf32 issues at half the f16 rate).
    The measured cuBLAS TF32 8192^3 figure (profiles/tf32_peak.json, ~0.43x
    bf16 on this pool) is reported beside it, not used as the denominator:
    our 3xTF32 GEMMs run faster than a third of it."""
    try:
        cublas = float(json.loads(TF32_PEAK.read_text())["tf32"]["sustained_tflops"])
    except Exception:
        cublas = None
    return bf16_sustained / 2.0, "MEASURED_PEAKS bf16 sustained / 2", cublas


def gemm_flops_per_step(cfg, T, S):
    """Algorithmic 2*M*N*K flops of one HVP's GEMM chain:
    8 products per weight matrix per token (1 primal, 2 tangent forward; 1
    adjoint, 2 adjoint-tangent, 2 Hv backward) and 18 S x S x dh products per
    head for attention (no causal halving counted)."""
    L, d, ff, V, H = cfg["n_layer"], cfg["d"], cfg["ff"], cfg["vocab"], cfg["n_head"]
    n_mm = L * (3 * d * d + d * d + 2 * d * ff) + V * d
    attn = L * 18 * 2 * (T // S) * H * S * S * (d // H)
    return 8 * 2 * n_mm * T + attn


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU side
def _hvp_seconds(o, cfg, S):
    th = o.gpt_init(cfg, 0, 0.0, 0.0, prec=0)
    tok, tgt = o.gpt_batch(cfg, 1, S)
    v = o.draw_probe(th.size, 7, 1, prec=0)
    t0 = time.perf_counter()
    o.gpt_hvp(cfg, th, tok, tgt, 1, S, v)
    return time.perf_counter() - t0


def cpu_c2_step(B, S, k_mid, seqs=(8, 64), full_recurrence=True):
    """CPU seconds of one C2 Lanczos step, EXTRAPOLATED from bounded samples:
    * HVP leg (the oracle's f64 restatement of the Graph HVP -- the reference
      has no HVP of its own): one sequence of the full GPT-2-small
      model at each length in `seqs`, fitted with t = c0 + k * F(S), F the
      algorithmic flops of that sequence (gemm_flops_per_step: 16 N_mm S for
      the weight products + 36 L H S^2 dh for attention, so the S^2 term is
      carried by the model, not by a fit of noisy small-S timings) and c0 the
      token-independent part (weight-sized tape work); evaluated at B
      sequences of length S: c0 + k * F(B x S);
    * recurrence leg (the compiled REFERENCE's own dot/axpy/scale through its
      WorkerPool on all host cores, oracle/_ref): one step's recurrence + 2x CGS
      at the full P (or P/8, scaled x8), timed at j = 0 and j = 2 stored
      columns, linear in j."""
    from oracle.pyoracle import Oracle, Reference, nthreads
    o = Oracle()
    cfg = GPT2_SMALL
    ts = [_hvp_seconds(o, cfg, q) for q in seqs]
    F = [gemm_flops_per_step(cfg, q, q) for q in seqs]
    k = max((ts[-1] - ts[0]) / (F[-1] - F[0]), 0.0)
    c0 = max(ts[0] - k * F[0], 0.0)
    t_hvp = c0 + k * gemm_flops_per_step(cfg, B * S, S)
    P = 124439808
    legs = {"hvp": {"kind": "port", "seconds": t_hvp, "c0_s": c0, "s_per_tflop": k * 1e12,
                    "sample": f"oracle f64 HVP, GPT-2-small, 1 sequence at S={list(seqs)} -> "
                              f"{[round(t, 2) for t in ts]} s, t = c0 + k*flops(S), evaluated at {B}x{S} tokens"}}
    try:
        r = Reference()
        w = nthreads()
        P_rec = P if full_recurrence else P // 8
        t_j0 = r.time_recurrence(P_rec, w, 0, 1)
        t_j2 = r.time_recurrence(P_rec, w, 2, 1)
        t_rec = (t_j0 + (t_j2 - t_j0) / 2.0 * k_mid) * (P / P_rec)
        legs["recurrence"] = {"kind": "reference", "seconds": t_rec,
                              "sample": f"reference dot/axpy/scale (oracle/_ref WorkerPool, {w} workers) at P={P_rec}, "
                                        f"j=0 ({t_j0:.2f} s) and j=2 ({t_j2:.2f} s), linear to j={k_mid}"
                                        + ("" if full_recurrence else f", x{P // P_rec} to P={P}")}
    except Exception as exc:  # compiled reference unavailable: the oracle's port of the same primitives
        x1 = o.draw_probe(P // 8, 1, 1, prec=0)
        y1 = o.draw_probe(P // 8, 2, 1, prec=0)
        t0 = time.perf_counter()
        o.dot(x1, y1)
        o.axpy(-0.5, x1, y1, 0)
        per_op = (time.perf_counter() - t0) / 2.0 * 8
        t_rec = per_op * (5 + 4 * k_mid)
        legs["recurrence"] = {"kind": "port", "seconds": t_rec, "sample": f"oracle dot/axpy at P/8 x8 ({exc})"[:200]}
    sec = t_hvp + legs["recurrence"]["seconds"]
    return sec, legs


def cpu_baseline_c2(B, S, k_mid):
    from oracle.pyoracle import nthreads
    sec, legs = cpu_c2_step(B, S, k_mid, seqs=(8, 32), full_recurrence=False)
    return {"value": 1.0 / sec, "unit": "steps/s", "cores": nthreads(), "kind": "port", "extrapolated": True,
            "cpu_model": cpu_model(), "legs": legs,
            "sample": "one C2 step extrapolated from bounded samples: " + legs["hvp"]["sample"] + "; "
                      + legs["recurrence"]["sample"]}


def cpu_c1_run():
    """C1 in full on the CPU: the oracle's Lanczos restatement over its own
    Graph HVP, 1 Rademacher probe x 32 steps, full reorth, f32 vectors."""
    from oracle.pyoracle import Oracle
    o = Oracle()
    th = o.gpt_init(C1_MODEL, 0, 0.0, 0.0, prec=0)
    tok, tgt = o.gpt_batch(C1_MODEL, 4, 32)
    t0 = time.perf_counter()
    r = o.lanczos_gpt(C1_MODEL, th, tok, tgt, 4, 32, 32, reorth=True, seed=42, dist=1, prec=0, hvp_prec=1)
    sec = time.perf_counter() - t0
    return sec / len(r["alphas"]), len(r["alphas"])


def run_reference(args):
    """--impl reference: the reference CPU path on the host cores, same
    metric/config as the GPU arm. C1 is timed in full; C2 is one step
    extrapolated from bounded samples (extrapolated: true). Never imports the
    product package."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.pyoracle import nthreads
    cfgd = workload_config(args)
    if args.workload == "c1":
        per_step, n = cpu_c1_run()
        sec, extrap = per_step, False
        cpu = {"kind": "port", "cores": nthreads(), "extrapolated": False, "cpu_model": cpu_model(),
               "sample": f"C1 in full: oracle Lanczos restatement over its Graph HVP, {n} steps, full reorth, "
                         f"{per_step * n:.2f} s"}
        n_steps = n
    else:
        k_mid = args.k_max // 2  # the GPU arm's timed window is centred on column k_max/2
        sec, legs = cpu_c2_step(args.batch, args.seq, k_mid, seqs=(8, 128), full_recurrence=True)
        extrap = True
        cpu = {"kind": "port", "cores": nthreads(), "extrapolated": True, "cpu_model": cpu_model(), "legs": legs,
               "sample": "one C2 step extrapolated from bounded samples: " + legs["hvp"]["sample"] + "; "
                         + legs["recurrence"]["sample"]}
        n_steps = 1
    val = 1.0 / sec
    cpu["value"] = val
    cpu["unit"] = "steps/s"
    line = {"metric": METRIC, "value": val, "unit": "steps/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": n_steps, "steps_requested": args.steps, "warmup": 0, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (HVP) / f32 vectors",
            "data": "synthetic", "extrapolated": extrap, "config": cfgd, "cpu_baseline": cpu,
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU side
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2505_11564_b200 as sd
    from paper_2505_11564_b200 import gpt
    from paper_2505_11564_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    c1, c3 = args.workload == "c1", args.workload == "c3"
    # N > 1: C3 is data-sharded (the global batch over the ranks, Hv summed);
    # C1/C2 -- one B200 each by BASELINE -- are SLQ jobs of independent probe
    # chains, so their ranks run disjoint probes with no collective on the data
    # path (--partition data runs the data-sharded variant instead)
    partition = args.partition or ("data" if c3 else "probes")
    probes = world > 1 and partition == "probes"
    dworld, drank = (1, 0) if probes else (world, rank)
    use_comm = (world > 1 and not probes) or args.comm
    if world > 1 or args.comm:
        if world == 1:  # --comm: the multi-rank code path on one rank (NCCL, no peers)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29541")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = C1_MODEL if c1 else (C3_MODEL if c3 else GPT2_SMALL)
    B, S = (4, 32) if c1 else ((32, 2048) if c3 else (args.batch, args.seq))
    k_max = 32 if c1 else args.k_max
    if B % dworld:
        raise SystemExit(f"global batch {B} not divisible by {dworld} ranks")
    b_loc = B // dworld
    T_glob = B * S
    tok_all, tgt_all = gpt.synthetic_tokens(cfg["vocab"], B, S, seed=1)
    sl = slice(drank * b_loc * S, (drank + 1) * b_loc * S)
    if c3:  # b_loc sequences as micro-batches of one sequence, layers recomputed in the backward
        eng = gpt.GptHvp(cfg, 1, S, init_seed=0, tokens=tok_all[sl], targets=tgt_all[sl], loss_scale=1.0 / T_glob,
                         micro_batches=b_loc, recompute=args.c3_recompute)
    else:
        eng = gpt.GptHvp(cfg, b_loc, S, init_seed=0, tokens=tok_all[sl], targets=tgt_all[sl],
                         loss_scale=1.0 / T_glob)
    comm = sd.nccl_comm() if use_comm else None
    P = eng.P
    # N > 1: Lanczos vectors parameter-sharded over the ranks (split_evenly);
    # each apply all-gathers q, runs the rank's batch HVP and reduce-scatters Hv
    layout = sd.split_evenly(P, dworld) if use_comm else None
    op = eng.operator(comm, layout=layout)
    P_local = (layout.shard_bounds[drank][1] - layout.shard_bounds[drank][0]) if layout else P
    reduction = sd.REDUCE_TREE if args.reduction == "tree" else sd.REDUCE_ORDERED
    reorth = sd.REORTH_SELECTIVE if (c3 and args.c3_reorth == "selective") else sd.REORTH_FULL
    window = args.window if reorth == sd.REORTH_SELECTIVE else 0
    lcfg = lambda seed: sd.LanczosConfig(k_max=k_max, reorthogonalize=reorth, prec=sd.F32,  # noqa: E731
                                         probe=sd.ProbeSpec(seed=seed, distribution=sd.RADEMACHER),
                                         reduction=reduction, selective_window=window)
    # probe chains: seeds base, base + 1, ...; with probe partitioning rank r
    # takes seeds base + r, base + r + N, ... (its share of the SLQ job's probes)
    first_seed, pstride = probe_seed_plan(42 if c1 else 0, rank, world, probes)
    state = {"probe": first_seed, "L": None, "ws": None}

    def new_chain():
        if state["L"] is not None:
            state["L"].close()
        state["L"] = sd.Lanczos(op, lcfg(state["probe"]), layout=layout, comm=comm, workspace=state["ws"])
        state["ws"] = state["L"].workspace
        state["probe"] += pstride

    def step():
        if state["L"] is None or state["L"].done:
            new_chain()
        state["L"].step()

    new_chain()
    # untimed: W warm-up steps, then advance the chain so the timed window is
    # centred on k_max/2 -- its mean reorthogonalisation width equals that of
    # a whole k_max chain (full reorth cost grows linearly with the column)
    advance = max(0, k_max // 2 - args.steps // 2 - args.warmup) if args.steps < k_max else 0
    for _ in range(args.warmup + advance):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    L0 = lib()
    check = sd._lib.check
    launches0 = L0.sd_launch_count()
    j_first = state["L"].result().alphas.size + 1
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    launches = L0.sd_launch_count() - launches0
    res = state["L"].result()
    j_last = res.alphas.size
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    # whole job: every rank advanced its own chain (probe partitioning) or all
    # ranks advanced the one sharded chain together
    value = (world if probes else 1) * 1000.0 / ms_step

    # ---- e2e: the public step API with host buffers, every step: H2D of the
    # step's batch tokens (pinned) + Lanczos step + D2H of (alpha, beta)
    tok_pin = torch.from_numpy(np.ascontiguousarray(tok_all[sl])).pin_memory()
    tgt_pin = torch.from_numpy(np.ascontiguousarray(tgt_all[sl])).pin_memory()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    # the e2e window sits at the same reorthogonalisation width as the timed
    # window (full-reorth cost grows with the column): the timed chain's probe
    # is restarted and advanced, untimed, to e2e_steps steps centred on the
    # timed window's centre
    state["probe"] -= pstride
    new_chain()
    centre = (j_first + j_last) // 2
    for _ in range(max(0, centre - e2e_steps // 2 - 1)):
        step()
    e2e_first = state["L"].result().alphas.size + 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(e2e_steps):
        eng.set_batch(tok_pin.numpy(), tgt_pin.numpy(), 1.0 / T_glob)
        step()
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    # ---- profiled pass (separate from the headline): CUDA events around every
    # GEMM launch give the GEMM share of the step and its TF/s
    prof_steps = max(1, min(args.profile_steps, k_max - 2))
    torch.cuda.synchronize()
    check(L0.sd_gemm_profile_begin())
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for _ in range(prof_steps):
        step()
    p1.record()
    torch.cuda.synchronize()
    g_ms, g_fl, g_n = C.c_double(), C.c_double(), C.c_uint64()
    check(L0.sd_gemm_profile_end(C.byref(g_ms), C.byref(g_fl), C.byref(g_n)))
    prof_ms = p0.elapsed_time(p1)

    hbm, bf16, basis = peaks()
    tf32, tf32_basis, cublas_tf32 = tf32_peak(bf16)
    tc_peak = tf32 / 3.0  # 3xTF32: 3 tf32 MMAs per algorithmic product
    achieved = g_fl.value / (g_ms.value * 1e-3) / 1e12 if g_ms.value > 0 else 0.0
    traffic = alg_bytes = None
    if TRAFFIC_FILE.exists() and not c1 and not c3:
        try:
            tj = json.loads(TRAFFIC_FILE.read_text())
            traffic, alg_bytes = tj.get("bytes_per_launch"), tj.get("algorithmic_bytes_per_launch")
        except Exception:
            traffic = None
    k_mid = 0.5 * (j_first + j_last)
    # Lanczos bytes per step: tree mode 4 P (3 j + 8) (3 GEMV passes over j
    # columns + r, scale), ordered mode 4 P (7 + 3 j)
    j_eff = min(k_mid, window) if window else k_mid
    lanczos_bytes = 4.0 * P_local * ((3 * j_eff + 8) if reduction == sd.REDUCE_TREE else (7 + 3 * j_eff))
    step_roof_ms = gemm_flops_per_step(cfg, B * S, S) / dworld / (tc_peak * 1e12) * 1e3 + lanczos_bytes / (hbm * 1e9) * 1e3
    cfgd = workload_config(args)
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if probes else "strong",
        "vs_baseline": None, "dtype": "f32 (3xTF32 tensor-core GEMMs, fp32 storage, f64 Lanczos scalars)",
        "data": "synthetic (counter-keyed tokens, random-init weights)",
        "config": cfgd,
        "run": {"reorth_columns_timed": [j_first, j_last], "untimed_advance_steps": advance,
                "reduction": args.reduction,
                "parallelism": (f"{world} ranks x independent probe chains (no data-path collective)" if probes else
                                f"dp{world} batch x {world}-way sharded Lanczos (all-gather q, reduce-scatter Hv)"
                                if layout is not None else "dp1"),
                "l2": ("C1 fits in L2 (226 KB vectors)" if c1 else
                       "inputs larger than L2 (Lanczos vectors >= 0.5 GB, activations >= 10 GB)"),
                "memory_gb": {"hvp_workspace": eng.workspace.numel() / 1e9,
                              "lanczos_workspace": state["ws"].numel() / 1e9,
                              "device_peak": torch.cuda.max_memory_allocated() / 1e9}},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                     "frac": achieved / tc_peak if tc_peak else None, "traffic": traffic,
                     "algorithmic_bytes": alg_bytes,
                     "traffic_source": "profiles/r02_gemm_traffic.json (ncu dram bytes per GEMM launch, one HVP)",
                     "kernel": "k_gemm_pair + k_gemm_tf32 (3xTF32 tcgen05), all GEMM launches of the step",
                     "peak_note": f"3xTF32 roofline = {tf32_basis} ({basis}) = {tf32:.1f} TF/s / 3 (passes); "
                                  + (f"vs measured cuBLAS TF32 sustained {cublas_tf32:.1f} / 3 = "
                                     f"{cublas_tf32 / 3:.1f} TF/s the frac is {achieved / (cublas_tf32 / 3):.3f}"
                                     if cublas_tf32 else "no cuBLAS TF32 measurement"),
                     "measured_in": f"separate profiled pass of {prof_steps} steps (events around every GEMM)",
                     "gemm_share_of_step": (g_ms.value / prof_ms) if prof_ms else None,
                     "gemm_launches_per_step": int(g_n.value) / prof_steps},
        "roofline_step": {"bound": "tensor+hbm", "roofline_ms": step_roof_ms, "measured_ms": ms_step,
                          "frac": step_roof_ms / ms_step, "lanczos_bytes": lanczos_bytes, "hbm_peak_gbs": hbm},
        "e2e": {"value": (world if probes else 1) * 1000.0 / e2e_ms, "unit": "steps/s", "h2d_bytes_per_step": int(2 * tok_pin.numel() * 4),
                "d2h_bytes_per_step": 16, "steps": e2e_steps,
                "reorth_columns": [e2e_first, e2e_first + e2e_steps - 1]},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "lanczos_phase_ms_total": {"apply": res.ms_apply, "recurrence": res.ms_recurrence, "reorth": res.ms_reorth},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not c3:
        try:
            if c1:
                from oracle.pyoracle import nthreads
                per_step, n = cpu_c1_run()
                line["cpu_baseline"] = {"value": 1.0 / per_step, "unit": "steps/s", "cores": nthreads(), "kind": "port",
                                        "extrapolated": False, "cpu_model": cpu_model(),
                                        "sample": f"C1 in full: oracle Lanczos over its Graph HVP, {n} steps"}
            else:
                line["cpu_baseline"] = cpu_baseline_c2(B, S, int(k_mid))
        except Exception as exc:  # the CPU leg must not sink the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    state["L"].close()
    if comm is not None:
        comm.close()
    if world > 1 or args.comm:
        dist.destroy_process_group()


# ------------------------------------------------- pipeline workloads (C4/C5)
PIPE_WORKLOADS = {
    # BASELINE configs[3]: 7B Llama-style decoder, parameter-sharded Lanczos vectors,
    # scalar-dot allreduce, selective reorth (window of the 8 most recent columns)
    "c4": dict(model="LLAMA2_7B", bf16=0, flags=0, reorth="selective", window=8, k_max=32),
    # BASELINE configs[4]: 70B architecture, bf16 weights / fp32 Lanczos, 3-term recurrence
    "c5": dict(model="LLAMA_70B", bf16=1, flags=3, reorth="none", window=0, k_max=10),
}


def run_pipeline_workload(args):
    """C4/C5: pipeline-parallel HVP over the N ranks (stage r = layers
    split_evenly(n_layer, N)[r]), Lanczos vectors sharded by the stages'
    parameter slices, M micro-batches of 1 x seq tokens per HVP on the 1F1B
    schedule. --layers shrinks the depth (to run the path on fewer GPUs)."""
    import torch
    import torch.distributed as dist

    import paper_2505_11564_b200 as sd
    from paper_2505_11564_b200 import gpt
    from paper_2505_11564_b200._lib import lib

    wl = PIPE_WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29543")
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    comm = sd.nccl_comm()
    cfg = dict(getattr(gpt, wl["model"]), bf16_weights=wl["bf16"])
    if args.layers:
        cfg["n_layer"] = args.layers
    M, S = args.micro_batches, args.seq
    l0, l1 = gpt.pipeline_layers(cfg["n_layer"], world)[rank]
    b, e = gpt.stage_params(cfg, l0, l1)
    theta = gpt.init_params_range(cfg, b, e, init_seed=0)
    tok, tgt = gpt.synthetic_tokens(cfg["vocab"], M, S, seed=1)
    st = gpt.GptStage(cfg, 1, S, M, l0, l1, theta, n_sets=min(M, world - rank), tokens=tok, targets=tgt,
                      recompute=bool(wl["flags"] & 1), probe_residual=not (wl["flags"] & 2))
    layout = gpt.pipeline_layout(cfg, world)
    reorth = {"selective": sd.REORTH_SELECTIVE, "none": sd.REORTH_NONE}[wl["reorth"]]
    k_max = max(args.k_max if args.k_max != 100 else wl["k_max"], args.steps + args.warmup + 1)
    lc = sd.LanczosConfig(k_max=k_max + args.profile_steps, reorthogonalize=reorth, prec=sd.F32,
                          probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER), selective_window=wl["window"],
                          reduction=sd.REDUCE_TREE if args.reduction == "tree" else sd.REDUCE_ORDERED)
    L = sd.Lanczos(st.operator(comm), lc, layout=layout, comm=comm)
    for _ in range(args.warmup):
        L.step()
    torch.cuda.synchronize()
    dist.barrier()
    L0 = lib()
    check = sd._lib.check
    launches0 = L0.sd_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            L.step()
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    launches = L0.sd_launch_count() - launches0
    # GEMM share / TF/s from a separate profiled pass (the timed loop carries no events)
    check(L0.sd_gemm_profile_begin())
    for _ in range(max(1, args.profile_steps)):
        L.step()
    torch.cuda.synchronize()
    g_ms, g_fl, g_n = C.c_double(), C.c_double(), C.c_uint64()
    check(L0.sd_gemm_profile_end(C.byref(g_ms), C.byref(g_fl), C.byref(g_n)))
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    hbm, bf16, basis = peaks()
    tf32, tf32_basis, _ = tf32_peak(bf16)
    achieved = g_fl.value / (g_ms.value * 1e-3) / 1e12 if g_ms.value > 0 else 0.0
    line = {
        "metric": METRIC, "value": 1000.0 / ms_step, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (3xTF32 GEMMs" + (", bf16-valued weights" if wl["bf16"] else "") + ")",
        "data": "synthetic (counter-keyed tokens, random-init weights)",
        "config": {"workload": f"BASELINE {args.workload.upper()}: pipeline-parallel HVP, {world} stage(s)",
                   "model": wl["model"], "n_layer": cfg["n_layer"], "params": gpt.param_count(cfg),
                   "micro_batches": M, "seq_len": S, "tokens_per_hvp": M * S, "reorth": wl["reorth"],
                   "k_max": k_max, "engine_flags": wl["flags"], "parallelism": f"pp{world}",
                   "reduction": args.reduction,
                   "bubble_bound": M / (M + world - 1)},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": tf32 / 3.0, "unit": "TFLOP/s",
                     "frac": achieved / (tf32 / 3.0), "traffic": None,
                     "kernel": "all GEMM launches of rank 0's stage", "peak_note": f"{tf32_basis} ({basis}) / 3"},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    L.close()
    comm.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--k-max", type=int, default=100)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--comm", action="store_true", help="use the NCCL/sharded path even on one rank")
    ap.add_argument("--partition", default=None, choices=["probes", "data"],
                    help="N > 1: probes (independent probe chains per rank; default for c1/c2) or data "
                         "(data-sharded HVP + parameter-sharded Lanczos; default for c3)")
    ap.add_argument("--c3-reorth", default="selective", choices=["selective", "full"],
                    help="C3: selective (window --window, fits one GPU) or full (sharded basis, N >= 4)")
    ap.add_argument("--window", type=int, default=16, help="selective reorth window (C3)")
    ap.add_argument("--c3-recompute", action="store_true",
                    help="C3: keep only layer inputs, re-run layers in the backward (less memory, ~1/3 more flops)")
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="c2 (default, the metric's config), c1 (BASELINE configs[0]) or the C4/C5 "
                         "pipeline-parallel workloads")
    ap.add_argument("--reduction", default="tree", choices=["tree", "ordered"],
                    help="Lanczos reductions: tree (fused GEMV passes, fixed-order tree sums; HVP configs) or "
                         "ordered (the reference's 1024-block fold, bitwise parity mode)")
    ap.add_argument("--profile-steps", type=int, default=3, help="steps of the separate GEMM-profiled pass")
    ap.add_argument("--layers", type=int, default=0, help="C4/C5: override the depth (0 = the model's)")
    ap.add_argument("--micro-batches", type=int, default=32, help="C4/C5: micro-batches per HVP")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload in ("c4", "c5"):
        run_pipeline_workload(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
