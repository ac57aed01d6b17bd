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

N > 1 (torchrun, one rank per GPU): strong scaling of the same global batch,
data-sharded HVP (each rank B/N sequences) with an NCCL all-reduce of Hv;
Lanczos vectors are replicated (identical on every rank after the
all-reduce), so the recurrence needs no further collective.
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
TRAFFIC_FILE = ROOT / "profiles" / "gemm_traffic.json"
METRIC = "Lanczos steps/sec (HVP+reorth) at 1/2/4/8 B200; HVP/Lanczos roofline fraction"


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
def cpu_sample(cfg, B, S, k_mid, reference_primitives: bool):
    """Bounded CPU sample of one step of the same workload: the HVP of the
    full GPT-2-small model on 1 x S_s tokens (oracle restatement, f64, all
    host cores), scaled linearly to B x S tokens, plus the Lanczos recurrence
    and 2x CGS at full P measured with the compiled reference's own
    dot/axpy/scale (oracle/_ref) at j = 0 and j = 2 and extrapolated linearly
    to j = k_mid."""
    from oracle.pyoracle import Oracle, Reference, nthreads
    o = Oracle()
    S_s = 16
    th = o.gpt_init(cfg, 0, 0.0, 0.0, prec=0)
    tok, tgt = o.gpt_batch(cfg, 1, S_s)
    v = o.draw_probe(th.size, 7, 1, prec=0)
    t0 = time.perf_counter()
    o.gpt_hvp(cfg, th, tok, tgt, 1, S_s, v)
    t_hvp = (time.perf_counter() - t0) * (B * S) / S_s
    P = th.size
    del th, v
    kind = "port"
    if reference_primitives:
        try:
            r = Reference()
            w = nthreads()
            t_j0 = r.time_recurrence(P, w, 0, 1)
            t_j2 = r.time_recurrence(P, w, 2, 1)
            t_rec = t_j0 + (t_j2 - t_j0) / 2.0 * k_mid
            kind = "reference"
        except Exception:
            reference_primitives = False
    if not reference_primitives:
        x = o.draw_probe(P, 1, 1, prec=0)
        y = o.draw_probe(P, 2, 1, prec=0)
        t0 = time.perf_counter()
        o.dot(x, y)
        o.axpy(-0.5, x, y, 0)
        per_op = (time.perf_counter() - t0) / 2.0
        t_rec = per_op * (5 + 4 * k_mid)
    sec = t_hvp + t_rec
    return {"value": 1.0 / sec, "unit": "steps/s", "cores": nthreads(), "kind": kind,
            "sample": (f"oracle f64 HVP of the full model on 1x{S_s} tokens scaled x{B * S // S_s} to {B}x{S}; "
                       f"recurrence + 2xCGS at full P={P} ({'reference dot/axpy/scale' if kind == 'reference' else 'oracle port'})"
                       f" at j=0,2 extrapolated to j={k_mid}"),
            "hvp_s": t_hvp, "recurrence_s": t_rec}


def run_reference(args):
    """--impl reference: the reference CPU path (compiled reference primitives +
    oracle HVP restatement; the reference has no HVP) timed on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2505_11564_b200.gpt import GPT2_SMALL
    cfg = GPT2_SMALL
    k_mid = args.k_max // 2  # same mean reorth width as the GPU arm's timed window
    # each reference "step" is one bounded CPU sample (~1 min on 8 cores); at
    # most two are run so the arm ends within a few minutes
    n = max(1, min(args.steps, 2))
    steps = [cpu_sample(cfg, args.batch, args.seq, k_mid, True) for _ in range(n)]
    sec = float(np.mean([1.0 / s["value"] for s in steps]))
    val = 1.0 / sec
    base = steps[-1]
    line = {"metric": METRIC, "value": val, "unit": "steps/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": n, "steps_requested": args.steps, "warmup": 0, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "gpt2-small 124M, synthetic tokens, batch 8x1024, full reorth",
                       "global_batch": args.batch, "seq_len": args.seq, "k_mid": k_mid},
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": base["cores"], "kind": base["kind"],
                             "sample": base["sample"]},
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
    use_comm = world > 1 or args.comm
    if use_comm:
        if world == 1:  # --comm: the multi-rank code path on one rank (NCCL, no peers)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29541")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = gpt.GPT2_SMALL
    B, S = args.batch, args.seq
    if B % world:
        raise SystemExit(f"global batch {B} not divisible by {world} ranks")
    b_loc = B // world
    T_glob = B * S
    tok_all, tgt_all = gpt.synthetic_tokens(cfg["vocab"], B, S, seed=1)
    sl = slice(rank * b_loc * S, (rank + 1) * b_loc * S)
    eng = gpt.GptHvp(cfg, b_loc, S, init_seed=0, tokens=tok_all[sl], targets=tgt_all[sl], loss_scale=1.0 / T_glob)
    comm = sd.nccl_comm() if use_comm else None
    P = eng.P
    # N > 1: Lanczos vectors parameter-sharded over the ranks (split_evenly);
    # each apply all-gathers q, runs the rank's batch HVP and reduce-scatters Hv
    layout = sd.split_evenly(P, world) if use_comm else None
    op = eng.operator(comm, layout=layout)
    P_local = (layout.shard_bounds[rank][1] - layout.shard_bounds[rank][0]) if layout else P
    lcfg = lambda seed: sd.LanczosConfig(k_max=args.k_max, reorthogonalize=sd.REORTH_FULL, prec=sd.F32,  # noqa: E731
                                         probe=sd.ProbeSpec(seed=seed, distribution=sd.RADEMACHER))
    ws_bytes = None
    state = {"probe": 0, "L": None, "ws": None, "done_probes": 0, "alphas": []}

    def new_chain():
        if state["L"] is not None:
            res = state["L"].result()
            state["alphas"].append(res.alphas)
            state["L"].close()
        state["L"] = sd.Lanczos(op, lcfg(state["probe"]), layout=layout, comm=comm, workspace=state["ws"])
        state["ws"] = state["L"].workspace
        state["probe"] += 1

    def step():
        if state["L"] is None or state["L"].done:
            new_chain()
        state["L"].step()

    new_chain()
    # untimed: W warm-up steps, then advance the chain so the timed window is
    # centred on k_max/2 -- its mean reorthogonalisation width equals that of
    # a whole k_max chain (full reorth cost grows linearly with the column)
    advance = max(0, args.k_max // 2 - args.steps // 2 - args.warmup) if args.steps < args.k_max else 0
    for _ in range(args.warmup + advance):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    L0 = lib()
    launches0 = L0.sd_launch_count()
    check = sd._lib.check
    check(L0.sd_gemm_profile_begin())
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
    g_ms, g_fl, g_n = C.c_double(), C.c_double(), C.c_uint64()
    check(L0.sd_gemm_profile_end(C.byref(g_ms), C.byref(g_fl), C.byref(g_n)))
    launches = L0.sd_launch_count() - launches0
    res = state["L"].result()
    j_last = res.alphas.size
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = 1000.0 / ms_step

    # ---- e2e: the public step API with host buffers, every step: H2D of the
    # step's batch tokens (pinned) + Lanczos step + D2H of (alpha, beta)
    tok_pin = torch.from_numpy(np.ascontiguousarray(tok_all[sl])).pin_memory()
    tgt_pin = torch.from_numpy(np.ascontiguousarray(tgt_all[sl])).pin_memory()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2 = time.perf_counter()
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
    del e2

    hbm, bf16, basis = peaks()
    tf32, tf32_basis, cublas_tf32 = tf32_peak(bf16)
    tc_peak = tf32 / 3.0  # 3xTF32: 3 tf32 MMAs per algorithmic product
    achieved = g_fl.value / (g_ms.value * 1e-3) / 1e12 if g_ms.value > 0 else 0.0
    traffic = None
    if TRAFFIC_FILE.exists():
        try:
            traffic = json.loads(TRAFFIC_FILE.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    k_mid = 0.5 * (j_first + j_last)
    lanczos_bytes = 4.0 * P_local * (7 + 3 * k_mid)
    step_roof_ms = gemm_flops_per_step(cfg, B * S, S) / world / (tc_peak * 1e12) * 1e3 + lanczos_bytes / (hbm * 1e9) * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (3xTF32 tensor-core GEMMs, fp32 storage, f64 Lanczos scalars)",
        "data": "synthetic (counter-keyed tokens, random-init GPT-2-small weights)",
        "config": {"workload": "BASELINE configs[1]: GPT-2-small shape 124M, batch 8x1024 tokens, "
                               "Rademacher probes, k_max=100, full reorth",
                   "model": "gpt2-small", "params": P, "global_batch": B, "seq_len": S, "k_max": args.k_max,
                   "reorth_columns_timed": [j_first, j_last], "untimed_advance_steps": advance,
                   "parallelism": (f"dp{world} batch x {world}-way sharded Lanczos (all-gather q, reduce-scatter Hv)"
                                   if layout is not None else "dp1"),
                   "l2": "inputs larger than L2 (0.5 GB Lanczos vectors, 45 GB activations)"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                     "frac": achieved / tc_peak if tc_peak else None, "traffic": traffic,
                     "kernel": "k_gemm_pair + k_gemm_tf32 (3xTF32 tcgen05), all GEMM launches of the step",
                     "peak_note": f"3xTF32 roofline = {tf32_basis} ({basis}) = {tf32:.1f} TF/s / 3 (passes); "
                                  + (f"vs measured cuBLAS TF32 sustained {cublas_tf32:.1f} / 3 = "
                                     f"{cublas_tf32 / 3:.1f} TF/s the frac is {achieved / (cublas_tf32 / 3):.3f}"
                                     if cublas_tf32 else "no cuBLAS TF32 measurement"),
                     "gemm_share_of_step": (g_ms.value / ms_total) if ms_total else None,
                     "gemm_launches": int(g_n.value)},
        "roofline_step": {"bound": "tensor+hbm", "roofline_ms": step_roof_ms, "measured_ms": ms_step,
                          "frac": step_roof_ms / ms_step, "lanczos_bytes": lanczos_bytes, "hbm_peak_gbs": hbm},
        "e2e": {"value": 1000.0 / e2e_ms, "unit": "steps/s", "h2d_bytes_per_step": int(2 * tok_pin.numel() * 4),
                "d2h_bytes_per_step": 16, "steps": e2e_steps},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "lanczos_phase_ms": {"apply": res.ms_apply, "recurrence": res.ms_recurrence, "reorth": res.ms_reorth},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_sample(cfg, B, S, int(k_mid), True)
        except Exception as exc:  # the CPU leg must not sink the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    state["L"].close()
    if comm is not None:
        comm.close()
    if use_comm:
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
    lc = sd.LanczosConfig(k_max=k_max, reorthogonalize=reorth, prec=sd.F32,
                          probe=sd.ProbeSpec(seed=0, distribution=sd.RADEMACHER), selective_window=wl["window"])
    L = sd.Lanczos(st.operator(comm), lc, layout=layout, comm=comm)
    for _ in range(args.warmup):
        L.step()
    torch.cuda.synchronize()
    dist.barrier()
    L0 = lib()
    check = sd._lib.check
    check(L0.sd_gemm_profile_begin())
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
    g_ms, g_fl, g_n = C.c_double(), C.c_double(), C.c_uint64()
    check(L0.sd_gemm_profile_end(C.byref(g_ms), C.byref(g_fl), C.byref(g_n)))
    launches = L0.sd_launch_count() - launches0
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
    ap.add_argument("--workload", default="c2", choices=["c2", "c4", "c5"],
                    help="c2 (default, the metric's config) or the C4/C5 pipeline-parallel workloads")
    ap.add_argument("--layers", type=int, default=0, help="C4/C5: override the depth (0 = the model's)")
    ap.add_argument("--micro-batches", type=int, default=32, help="C4/C5: micro-batches per HVP")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload != "c2":
        run_pipeline_workload(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
