"""MLP Hessian-vector products (SPEC.md:179 mlp(layer_widths), tanh hidden
layers, mse loss) on the sd_mlp_* C-ABI (csrc/sd_mlp.cu).

Mirrors the reference's hvp / batched_hvp surface: the flat
parameter vector is W_0 [w0 x w1] row-major, b_0, W_1, b_1, ... (declaration
order); batches are (x [n x w0], y [n x w_last]) and may be read
from the SPEC's columnar text format with `load_columnar`."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import ConfigError, check, lib
from .core import OperatorHandle

_ready = False


def _L():
    global _ready
    L = lib()
    if not _ready:
        u64p = C.POINTER(C.c_uint64)
        sig = {
            "sd_mlp_param_count": (C.c_uint64, [u64p, C.c_int]),
            "sd_mlp_create": (C.c_int, [u64p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
            "sd_mlp_set_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_float, C.c_void_p]),
            "sd_mlp_hvp": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
            "sd_mlp_last_loss": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
            "sd_mlp_destroy": (C.c_int, [C.c_void_p]),
            "sd_operator_mlp": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _ready = True
    return L


def _widths(widths):
    w = np.ascontiguousarray(widths, dtype=np.uint64)
    return w, w.ctypes.data_as(C.POINTER(C.c_uint64))


def param_count(widths) -> int:
    w, p = _widths(widths)
    return int(_L().sd_mlp_param_count(p, int(w.size)))


def load_columnar(path: str, n_targets: int = 1):
    """one sample per line, whitespace-separated features, the
    last column(s) the target. Returns float32 (x [n, f], y [n, n_targets])."""
    rows = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            try:
                rows.append([float(t) for t in s.split()])
            except ValueError as e:
                raise ConfigError(f"{path}:{ln}: not a number ({e})") from None
    if not rows:
        raise ConfigError(f"{path}: no samples")
    width = len(rows[0])
    if width <= n_targets or any(len(r) != width for r in rows):
        raise ConfigError(f"{path}: inconsistent sample dimensions")
    a = np.asarray(rows, dtype=np.float64)
    return a[:, :-n_targets].astype(np.float32), a[:, -n_targets:].astype(np.float32)


class MlpHvp:
    """HVP engine for one MLP on the current CUDA device."""

    def __init__(self, widths, theta: torch.Tensor, n_max: int, x=None, y=None, loss_scale: float | None = None,
                 stream=None):
        self.widths = [int(w) for w in widths]
        self.P = param_count(self.widths)
        assert theta.dtype == torch.float32 and theta.numel() == self.P and theta.is_contiguous() and theta.is_cuda
        self.theta = theta
        self.n_max = int(n_max)
        self.stream = stream or torch.cuda.current_stream()
        w, p = _widths(self.widths)
        self.h = C.c_void_p()
        check(_L().sd_mlp_create(p, int(w.size), self.n_max, theta.data_ptr(), C.c_void_p(self.stream.cuda_stream),
                                 C.byref(self.h)))
        self.n = 0
        if x is not None:
            self.set_batch(x, y, loss_scale)

    def set_batch(self, x, y, loss_scale: float | None = None):
        xa = np.ascontiguousarray(x, dtype=np.float32)
        ya = np.ascontiguousarray(y, dtype=np.float32).reshape(xa.shape[0], -1)
        if xa.ndim != 2 or xa.shape[1] != self.widths[0] or ya.shape[1] != self.widths[-1]:
            raise ConfigError("mlp batch shape does not match the widths")
        self._x, self._y = xa, ya
        self.n = xa.shape[0]
        scale = 1.0 / (self.n * self.widths[-1]) if loss_scale is None else loss_scale
        check(_L().sd_mlp_set_batch(self.h, xa.ctypes.data, ya.ctypes.data, self.n, scale,
                                    C.c_void_p(self.stream.cuda_stream)))

    def hvp(self, v: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        assert v.dtype == torch.float32 and v.numel() == self.P and v.is_contiguous()
        out = torch.empty_like(v) if out is None else out
        check(_L().sd_mlp_hvp(self.h, v.data_ptr(), out.data_ptr(), C.c_void_p(self.stream.cuda_stream)))
        return out

    def loss(self) -> float:
        x = C.c_double()
        check(_L().sd_mlp_last_loss(self.h, C.byref(x)))
        return x.value

    def operator(self, comm=None) -> OperatorHandle:
        h = C.c_void_p()
        check(_L().sd_operator_mlp(self.h, comm.handle if comm is not None else None, C.byref(h)))
        return OperatorHandle(self.P, f"mlp_hvp({self.widths})", h, keepalive=self)

    def close(self):
        if self.h:
            _L().sd_mlp_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def batched_hvp(engine: MlpHvp, batches, v: torch.Tensor) -> torch.Tensor:
    """PAPER.md Alg. 1 / SPEC.md:204-210: sum_b |B_b| u_b / N over (x, y)
    batches; each batch's mse is rescaled to 1/(N * w_last) so its Hv already
    carries the |B_b|/N weight, and the results are summed in batch order."""
    from .core import _scalar, _stream
    batches = list(batches)
    if not batches:
        raise ConfigError("batched_hvp needs at least one batch")
    N = sum(np.asarray(x).shape[0] for x, _ in batches)
    h = torch.zeros_like(v)
    tmp = torch.empty_like(v)
    one = _scalar(1.0, v.device)
    for x, y in batches:
        engine.set_batch(x, y, 1.0 / (N * engine.widths[-1]))
        engine.hvp(v, tmp)
        check(lib().sd_k_axpy(C.c_void_p(tmp.data_ptr()), C.c_void_p(h.data_ptr()), v.numel(),
                              C.c_void_p(one.data_ptr()), 1.0, 0, _stream()))
    return h
