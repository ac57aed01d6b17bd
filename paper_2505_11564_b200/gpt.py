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
                ("ctx", C.c_int), ("arch", C.c_int), ("rope_base", C.c_float), ("n_kv_head", C.c_int)]


ARCH_GPT2, ARCH_LLAMA = 0, 1
# BASELINE C4 (Llama-2-7B shape, MHA) -- the Llama-style decoder of this engine
LLAMA2_7B = dict(n_layer=32, d=4096, n_head=32, ff=11008, vocab=32000, ctx=4096, arch=ARCH_LLAMA, rope_base=10000)
# BASELINE C5 (R1-Distill-Llama-70B shape: 80L, d8192, ff28672, V128256, GQA 64/8)
LLAMA_70B = dict(n_layer=80, d=8192, n_head=64, ff=28672, vocab=128256, ctx=8192, arch=ARCH_LLAMA,
                 rope_base=500000, n_kv_head=8)


GPT2_SMALL = dict(n_layer=12, d=768, n_head=12, ff=3072, vocab=50257, ctx=1024)

_ready = False


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
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _ready = True
    return L


def _cfg(cfg: dict) -> GptConfig:
    return GptConfig(cfg["n_layer"], cfg["d"], cfg["n_head"], cfg["ff"], cfg["vocab"], cfg["ctx"],
                     cfg.get("arch", ARCH_GPT2), float(cfg.get("rope_base", 10000.0)), cfg.get("n_kv_head", 0))


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
    """HVP engine for one (batch, seq) shape on the current CUDA device."""

    def __init__(self, cfg: dict, batch: int, seq: int, init_seed: int = 0, gain_scale: float = 0.0,
                 bias_scale: float = 0.0, theta: torch.Tensor | None = None, tokens=None, targets=None,
                 seed_tok: int = 1, first_seq: int = 0, loss_scale: float | None = None, stream=None):
        self.cfg = dict(cfg)
        self.B, self.S = batch, seq
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
        nbytes = _L().sd_gpt_workspace_bytes(C.byref(self._c), batch, seq)
        if nbytes == 0:
            check(1)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.h = C.c_void_p()
        check(_L().sd_gpt_create(C.byref(self._c), batch, seq, theta.data_ptr(), self.workspace.data_ptr(), nbytes, s,
                                 C.byref(self.h)))
        if tokens is None:
            tokens, targets = synthetic_tokens(cfg["vocab"], batch, seq, seed_tok, first_seq)
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
