"""Python handle on the GPT HVP engine (sd_gpt_* of include/specden_b200.h).

``GptHvp`` owns the device parameters (torch, plumbing only), the engine
workspace, and the current batch; ``hvp`` runs PAPER.md Alg. 1 for one batch
(batch-size weighting across batches is ``batched_hvp``) and ``operator``
wraps the engine as the OperatorHandle the Lanczos engine drives.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import check, lib
from .core import OperatorHandle

_M64 = (1 << 64) - 1


class GptConfig(C.Structure):
    _fields_ = [("n_layer", C.c_int), ("d", C.c_int), ("n_head", C.c_int), ("ff", C.c_int), ("vocab", C.c_int),
                ("ctx", C.c_int), ("arch", C.c_int), ("rope_base", C.c_float), ("n_kv_head", C.c_int),
                ("bf16_weights", C.c_int)]


ARCH_GPT2, ARCH_LLAMA = 0, 1
# BASELINE C4 (Llama-2-7B shape, MHA) -- the Llama-style decoder of this engine
LLAMA2_7B = dict(n_layer=32, d=4096, n_head=32, ff=11008, vocab=32000, ctx=4096, arch=ARCH_LLAMA, rope_base=10000)
# BASELINE C5 (R1-Distill-Llama-70B shape: 80L, d8192, ff28672, V128256, GQA 64/8)
LLAMA_70B = dict(n_layer=80, d=8192, n_head=64, ff=28672, vocab=128256, ctx=8192, arch=ARCH_LLAMA,
                 rope_base=500000, n_kv_head=8)


GPT2_SMALL = dict(n_layer=12, d=768, n_head=12, ff=3072, vocab=50257, ctx=1024)

_ready = False
RECOMPUTE, NO_PROBE_RESIDUAL = 1, 2  # engine flags (sd_gpt_stage_create)


def _L():
    global _ready
    L = lib()
    if not _ready:
        cp = C.POINTER(GptConfig)
        sig = {
            "sd_gpt_param_count": (C.c_uint64, [cp]),
            "sd_gpt_param_layout": (C.c_int, [cp, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
            "sd_gpt_init_params": (C.c_int, [cp, C.c_uint64, C.c_double, C.c_double, C.c_void_p, C.c_void_p]),
            "sd_gpt_workspace_bytes": (C.c_uint64, [cp, C.c_int, C.c_int]),
            "sd_gpt_create": (C.c_int, [cp, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                        C.POINTER(C.c_void_p)]),
            "sd_gpt_set_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p]),
            "sd_gpt_hvp": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
            "sd_gpt_last_loss": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_void_p]),
            "sd_gpt_destroy": (C.c_int, [C.c_void_p]),
            "sd_operator_gpt": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
            "sd_operator_gpt_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
                                                  C.POINTER(C.c_uint64), C.POINTER(C.c_void_p)]),
            "sd_gpt_stage_workspace_bytes": (C.c_uint64, [cp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                          C.c_int]),
            "sd_gpt_stage_params": (C.c_int, [cp, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
            "sd_gpt_stage_create": (C.c_int, [cp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_void_p)]),
            "sd_gpt_stage_begin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
            "sd_gpt_stage_forward": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_void_p]),
            "sd_gpt_stage_backward": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p]),
            "sd_operator_gpt_pipeline": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
            "sd_gpt_init_params_range": (C.c_int, [cp, C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                                                   C.c_void_p, C.c_void_p]),
            "sd_pipeline_schedule": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_uint64,
                                               C.POINTER(C.c_uint64)]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _ready = True
    return L


def _cfg(cfg: dict) -> GptConfig:
    return GptConfig(cfg["n_layer"], cfg["d"], cfg["n_head"], cfg["ff"], cfg["vocab"], cfg["ctx"],
                     cfg.get("arch", ARCH_GPT2), float(cfg.get("rope_base", 10000.0)), cfg.get("n_kv_head", 0),
                     int(cfg.get("bf16_weights", 0)))


def param_count(cfg: dict) -> int:
    return int(_L().sd_gpt_param_count(C.byref(_cfg(cfg))))


def param_layout(cfg: dict):
    n = 4 + 12 * cfg["n_layer"]
    off, rows, cols = (np.zeros(n, np.uint64) for _ in range(3))
    kinds = np.zeros(n, np.int32)
    cnt = C.c_uint64()
    check(_L().sd_gpt_param_layout(C.byref(_cfg(cfg)), off.ctypes.data, rows.ctypes.data, cols.ctypes.data,
                                   kinds.ctypes.data, C.byref(cnt)))
    return [(int(off[i]), int(rows[i]), int(cols[i]), int(kinds[i])) for i in range(cnt.value)]


def _mix64(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(_M64)
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & np.uint64(_M64)
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & np.uint64(_M64)
    return z ^ (z >> np.uint64(31))


def synthetic_tokens(vocab: int, B: int, S: int, seed: int = 1, first_seq: int = 0):
    """Counter-keyed token streams (rng.hpp:50-52 uniform_index): sequence q is
    uniform_index(seed, q*(S+1) + s, V) for s in 0..S; inputs are its first S
    tokens, targets the next-token shift."""
    with np.errstate(over="ignore"):
        key = _mix64(np.uint64(seed))
        q = np.arange(first_seq, first_seq + B, dtype=np.uint64)[:, None]
        s = np.arange(S + 1, dtype=np.uint64)[None, :]
        ctr = q * np.uint64(S + 1) + s
        kc = _mix64(key ^ ((ctr * np.uint64(0x9E3779B97F4A7C15)) & np.uint64(_M64)))
        stream = (kc % np.uint64(vocab)).astype(np.int32)
    return np.ascontiguousarray(stream[:, :S]).reshape(-1), np.ascontiguousarray(stream[:, 1:]).reshape(-1)


class GptHvp:
    """HVP engine for one (batch, seq) shape on the current CUDA device.

    ``micro_batches`` = M runs the batch as M micro-batches of ``batch``
    sequences each (Alg. 1: Hv accumulated over the loader), so the
    workspace holds one micro-batch's activations; ``recompute`` keeps only
    each layer's input and re-runs the layer in the backward
    (SD_GPT_RECOMPUTE); ``probe_residual=False`` forms the probe's tf32
    residuals on chip (SD_GPT_NO_PROBE_RESIDUAL). Tokens are M * batch * seq."""

    def __init__(self, cfg: dict, batch: int, seq: int, init_seed: int = 0, gain_scale: float = 0.0,
                 bias_scale: float = 0.0, theta: torch.Tensor | None = None, tokens=None, targets=None,
                 seed_tok: int = 1, first_seq: int = 0, loss_scale: float | None = None, stream=None,
                 micro_batches: int = 1, recompute: bool = False, probe_residual: bool = True):
        self.cfg = dict(cfg)
        self.mb, self.M = batch, micro_batches
        self.B, self.S = batch * micro_batches, seq
        self._c = _cfg(cfg)
        self.P = param_count(cfg)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.current_stream()
        s = C.c_void_p(self.stream.cuda_stream)
        if theta is None:
            theta = torch.empty(self.P, dtype=torch.float32, device=self.device)
            check(_L().sd_gpt_init_params(C.byref(self._c), init_seed, gain_scale, bias_scale, theta.data_ptr(), s))
        assert theta.dtype == torch.float32 and theta.numel() == self.P and theta.is_contiguous()
        self.theta = theta
        self.flags = (RECOMPUTE if recompute else 0) | (0 if probe_residual else NO_PROBE_RESIDUAL)
        L_ = cfg["n_layer"]
        nbytes = _L().sd_gpt_stage_workspace_bytes(C.byref(self._c), batch, seq, micro_batches, 0, L_, 1, self.flags)
        self.h = C.c_void_p()
        if nbytes == 0:  # invalid shape: the create call raises the precise error class
            check(_L().sd_gpt_stage_create(C.byref(self._c), batch, seq, micro_batches, 0, L_, 1, self.flags, None,
                                           None, 0, s, C.byref(C.c_void_p())))
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        check(_L().sd_gpt_stage_create(C.byref(self._c), batch, seq, micro_batches, 0, L_, 1, self.flags,
                                       theta.data_ptr(), self.workspace.data_ptr(), nbytes, s, C.byref(self.h)))
        if tokens is None:
            tokens, targets = synthetic_tokens(cfg["vocab"], self.B, seq, seed_tok, first_seq)
        self.set_batch(tokens, targets, loss_scale)

    def set_batch(self, tokens, targets, loss_scale: float | None = None):
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        tgt = np.ascontiguousarray(targets, dtype=np.int32)
        assert tok.size == self.B * self.S == tgt.size
        self._tok, self._tgt = tok, tgt
        scale = 1.0 / tok.size if loss_scale is None else loss_scale
        check(_L().sd_gpt_set_batch(self.h, tok.ctypes.data, tgt.ctypes.data, scale,
                                    C.c_void_p(self.stream.cuda_stream)))

    def hvp(self, v: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        assert v.dtype == torch.float32 and v.numel() == self.P and v.is_contiguous()
        out = torch.empty_like(v) if out is None else out
        check(_L().sd_gpt_hvp(self.h, v.data_ptr(), out.data_ptr(), C.c_void_p(self.stream.cuda_stream)))
        return out

    def hvp_numpy(self, v) -> np.ndarray:
        vt = torch.tensor(np.asarray(v, np.float64), dtype=torch.float32, device=self.device)
        return self.hvp(vt).double().cpu().numpy()

    def loss(self) -> float:
        x = C.c_double()
        check(_L().sd_gpt_last_loss(self.h, C.byref(x), C.c_void_p(self.stream.cuda_stream)))
        return x.value

    def theta_numpy(self) -> np.ndarray:
        return self.theta.double().cpu().numpy()

    def tokens_numpy(self):
        return self._tok.astype(np.uint32), self._tgt.astype(np.uint32)

    def operator(self, comm=None, layout=None) -> OperatorHandle:
        """y = H x over this rank's batch, summed over `comm`'s ranks. With a
        `layout` the Lanczos vectors are parameter-sharded: x/y are this rank's
        shard, Hv is reduce-scattered (sd_operator_gpt_sharded)."""
        h = C.c_void_p()
        ch = comm.handle if comm is not None else None
        if layout is not None:
            b = (C.c_uint64 * len(layout.begins))(*layout.begins)
            e = (C.c_uint64 * len(layout.ends))(*layout.ends)
            check(_L().sd_operator_gpt_sharded(self.h, ch, b, e, C.byref(h)))
        else:
            check(_L().sd_operator_gpt(self.h, ch, C.byref(h)))
        return OperatorHandle(self.P, f"gpt_hvp(L={self.cfg['n_layer']},d={self.cfg['d']})", h, keepalive=self)

    def close(self):
        if self.h:
            _L().sd_gpt_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ pipeline stages
PIPE_F, PIPE_B, PIPE_SEND_F, PIPE_RECV_F, PIPE_SEND_B, PIPE_RECV_B, PIPE_GROUP_BEGIN, PIPE_GROUP_END = range(8)
PIPE_NAMES = ["F", "B", "SEND_F", "RECV_F", "SEND_B", "RECV_B", "GROUP_BEGIN", "GROUP_END"]


def stage_workspace_bytes(cfg: dict, micro_batch: int, seq: int, n_micro: int, layer_begin: int, layer_end: int,
                          n_sets: int, flags: int = 0) -> int:
    """Device workspace of one stage (host-side planning; no GPU needed)."""
    n = _L().sd_gpt_stage_workspace_bytes(C.byref(_cfg(cfg)), micro_batch, seq, n_micro, layer_begin, layer_end,
                                          n_sets, flags)
    if n == 0:
        check(3)
    return int(n)


def pipeline_schedule(n_stages: int, stage: int, n_micro: int):
    """1F1B schedule of one stage as [(kind, micro_batch)] (sd_pipeline_schedule; host only)."""
    n = C.c_uint64()
    check(_L().sd_pipeline_schedule(n_stages, stage, n_micro, None, 0, C.byref(n)))
    ops = np.zeros(2 * n.value, np.int32)
    check(_L().sd_pipeline_schedule(n_stages, stage, n_micro, ops.ctypes.data, n.value, C.byref(n)))
    return [(int(ops[2 * i]), int(ops[2 * i + 1])) for i in range(n.value)]


def pipeline_layers(n_layer: int, n_stages: int):
    """Contiguous layer ranges per stage: split_evenly over the layers
    (layout.hpp:59-72 semantics: the first n_layer % n_stages get one more)."""
    from .core import split_evenly
    lay = split_evenly(n_layer, n_stages)
    if len(lay.begins) != n_stages:
        raise ValueError("more pipeline stages than layers")
    return list(zip(lay.begins, lay.ends))


def stage_params(cfg: dict, layer_begin: int, layer_end: int):
    """[begin, end) of the stage's slice of the flat parameter vector."""
    b, e = C.c_uint64(), C.c_uint64()
    check(_L().sd_gpt_stage_params(C.byref(_cfg(cfg)), layer_begin, layer_end, C.byref(b), C.byref(e)))
    return int(b.value), int(e.value)


def init_params_range(cfg: dict, begin: int, end: int, init_seed: int = 0, gain_scale: float = 0.0,
                      bias_scale: float = 0.0, out: torch.Tensor | None = None) -> torch.Tensor:
    """Synthetic parameters of the flat range [begin, end) (a stage's slice),
    bit-identical to that slice of the full init."""
    if out is None:
        out = torch.empty(end - begin, dtype=torch.float32, device=torch.device("cuda", torch.cuda.current_device()))
    check(_L().sd_gpt_init_params_range(C.byref(_cfg(cfg)), init_seed, gain_scale, bias_scale, begin, end,
                                        out.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def pipeline_layout(cfg: dict, n_stages: int):
    """The Lanczos ShardLayout of a pipeline: shard r = stage r's parameters."""
    from .core import ShardLayout, validate_layout
    lay = ShardLayout(param_count(cfg), tuple(stage_params(cfg, a, b)
                                              for a, b in pipeline_layers(cfg["n_layer"], n_stages)))
    validate_layout(lay)
    return lay


class GptStage:
    """One pipeline stage (layers [layer_begin, layer_end)) of the Llama-style
    engine on the current device: stage-local theta (a slice of the flat
    parameters), n_micro micro-batches through n_sets activation sets."""

    def __init__(self, cfg: dict, micro_batch: int, seq: int, n_micro: int, layer_begin: int, layer_end: int,
                 theta_stage: torch.Tensor, n_sets: int | None = None, tokens=None, targets=None,
                 loss_scale: float | None = None, stream=None, recompute: bool = False,
                 probe_residual: bool = True):
        self.cfg = dict(cfg)
        self.B, self.S, self.M = micro_batch, seq, n_micro
        self.l0, self.l1 = layer_begin, layer_end
        self.n_sets = n_micro if n_sets is None else n_sets
        self._c = _cfg(cfg)
        self.P = param_count(cfg)
        self.begin, self.end = stage_params(cfg, layer_begin, layer_end)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.current_stream()
        assert theta_stage.dtype == torch.float32 and theta_stage.numel() == self.end - self.begin
        self.theta = theta_stage
        self.flags = (RECOMPUTE if recompute else 0) | (0 if probe_residual else NO_PROBE_RESIDUAL)
        nbytes = _L().sd_gpt_stage_workspace_bytes(C.byref(self._c), micro_batch, seq, n_micro, layer_begin,
                                                   layer_end, self.n_sets, self.flags)
        if nbytes == 0:  # invalid shape: the create call raises the precise error class
            check(_L().sd_gpt_stage_create(C.byref(self._c), micro_batch, seq, n_micro, layer_begin, layer_end,
                                           self.n_sets, self.flags, None, None, 0, self._s(),
                                           C.byref(C.c_void_p())))
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.h = C.c_void_p()
        check(_L().sd_gpt_stage_create(C.byref(self._c), micro_batch, seq, n_micro, layer_begin, layer_end,
                                       self.n_sets, self.flags, theta_stage.data_ptr(), self.workspace.data_ptr(),
                                       nbytes, self._s(), C.byref(self.h)))
        if tokens is None:
            tokens, targets = synthetic_tokens(cfg["vocab"], micro_batch * n_micro, seq)
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        tgt = np.ascontiguousarray(targets, dtype=np.int32)
        assert tok.size == n_micro * micro_batch * seq == tgt.size
        scale = 1.0 / tok.size if loss_scale is None else loss_scale
        check(_L().sd_gpt_set_batch(self.h, tok.ctypes.data, tgt.ctypes.data, scale, self._s()))

    def _s(self):
        return C.c_void_p(self.stream.cuda_stream)

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def begin_pass(self, v_stage: torch.Tensor, hv_stage: torch.Tensor):
        check(_L().sd_gpt_stage_begin(self.h, v_stage.data_ptr(), hv_stage.data_ptr(), self._s()))

    def forward(self, m: int, x_in=None, dx_in=None, x_out=None, dx_out=None):
        check(_L().sd_gpt_stage_forward(self.h, m, self._p(x_in), self._p(dx_in), self._p(x_out), self._p(dx_out),
                                        self._s()))

    def backward(self, m: int, gx_in=None, gdx_in=None, gx_out=None, gdx_out=None):
        check(_L().sd_gpt_stage_backward(self.h, m, self._p(gx_in), self._p(gdx_in), self._p(gx_out),
                                         self._p(gdx_out), self._s()))

    def loss(self) -> float:
        x = C.c_double()
        check(_L().sd_gpt_last_loss(self.h, C.byref(x), self._s()))
        return x.value

    def operator(self, comm) -> OperatorHandle:
        """Pipeline operator: comm rank r = this stage; x/y are the stage's slice."""
        h = C.c_void_p()
        check(_L().sd_operator_gpt_pipeline(self.h, comm.handle if comm is not None else None, C.byref(h)))
        return OperatorHandle(self.P, f"gpt_pipeline(L={self.cfg['n_layer']},stage={self.l0}-{self.l1})", h,
                              keepalive=self)

    def close(self):
        if self.h:
            _L().sd_gpt_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def batched_hvp(engines, v: torch.Tensor) -> torch.Tensor:
    """PAPER.md Alg. 1 lines 5-17: h = sum_b |B_b| u_b / N. Each engine's loss
    is rescaled to 1/N_tokens(total) so that its Hv already carries the
    |B_b|/N weight; the per-batch results are summed with the f32 axpy kernel."""
    from .core import _scalar, _stream
    tot = sum(e.B * e.S for e in engines)
    h = torch.zeros_like(v)
    tmp = torch.empty_like(v)
    one = _scalar(1.0, v.device)
    for e in engines:
        e.set_batch(e._tok, e._tgt, 1.0 / tot)
        e.hvp(v, tmp)
        check(lib().sd_k_axpy(C.c_void_p(tmp.data_ptr()), C.c_void_p(h.data_ptr()), v.numel(),
                              C.c_void_p(one.data_ptr()), 1.0, 0, _stream()))
    return h
