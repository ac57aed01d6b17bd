"""Host-side mirror of the reference's specden API (proj/include/specden/*.hpp,
SPEC.md) over the C-ABI of libspecden_b200.so.

Names, argument meaning and error behaviour follow the reference:
ShardLayout/split_evenly/validate_layout (layout.hpp), ShardedVector,
make_sharded, draw_probe, dot, norm2, axpy, scale, gather, scatter
(sharded.hpp), OperatorHandle + dense/wigner/spiked operators
(operators.hpp), and the SPEC-only lanczos_run / ritz_decompose /
smooth_density / average_spectra. Device memory is owned by torch tensors
(plumbing only); every floating-point op runs in the CUDA library.

A ShardedVector keeps one device tensor per shard. Several shards may live on
the same GPU (the reference's in-process WorkerPool emulation); scalar
reductions then exercise the same multi-rank ordered fold the NCCL path uses.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (ArgumentError, ConfigError, LayoutError, NumericalError, ProtocolError, StateError,  # noqa: F401
                   check, lib)

F32, F64 = 0, 1
GAUSSIAN, RADEMACHER, ONE_HOT, GAUSSIAN_DEVICE = 0, 1, 2, 3  # GAUSSIAN: bit-exact (host libm); _DEVICE: CUDA log/cos
REORTH_NONE, REORTH_FULL, REORTH_SELECTIVE = 0, 1, 2
REDUCE_ORDERED, REDUCE_TREE = 0, 1
_DTYPE = {F32: torch.float32, F64: torch.float64}


def parse_precision(s: str) -> int:
    """precision.hpp:30-34"""
    if s == "f32":
        return F32
    if s == "f64":
        return F64
    raise ConfigError(f"unknown precision '{s}' (expected f32 or f64)")


def unit_roundoff(prec: int) -> float:
    return 2.0 ** -24 if prec == F32 else 2.0 ** -53


def parse_probe_dist(s: str) -> int:
    """sharded.cpp:32-37"""
    try:
        return {"gaussian": GAUSSIAN, "rademacher": RADEMACHER, "one_hot": ONE_HOT}[s]
    except KeyError:
        raise ConfigError(f"unknown probe distribution '{s}'") from None


def _u64(xs):
    return (C.c_uint64 * len(xs))(*xs)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


# ------------------------------------------------------------------ layout
@dataclass(frozen=True)
class ShardLayout:
    """layout.hpp:18-43: contiguous half-open shards covering [0, total_dim)."""
    total_dim: int
    shard_bounds: tuple

    def worker_count(self) -> int:
        return len(self.shard_bounds)

    def owner(self, i: int) -> int:
        ends = _u64([e for _, e in self.shard_bounds])
        out = C.c_uint64()
        check(lib().sd_layout_owner(len(self.shard_bounds), ends, i, C.byref(out)))
        return out.value

    @property
    def begins(self):
        return [b for b, _ in self.shard_bounds]

    @property
    def ends(self):
        return [e for _, e in self.shard_bounds]


def validate_layout(l: ShardLayout) -> None:
    n = len(l.shard_bounds)
    check(lib().sd_validate_layout(l.total_dim, n, _u64(l.begins), _u64(l.ends)))


def split_evenly(dim: int, n: int) -> ShardLayout:
    if dim <= 0 or n <= 0:
        raise LayoutError("split_evenly needs dim > 0 and n > 0")
    m = min(dim, n)
    b = (C.c_uint64 * m)()
    e = (C.c_uint64 * m)()
    cnt = C.c_uint64()
    check(lib().sd_split_evenly(dim, n, b, e, C.byref(cnt)))
    return ShardLayout(dim, tuple((b[i], e[i]) for i in range(cnt.value)))


# ------------------------------------------------------------------ vectors
@dataclass
class ShardedVector:
    layout: ShardLayout
    prec: int
    shards: list = field(default_factory=list)

    def dim(self) -> int:
        return self.layout.total_dim


class WorkerPool:
    """In-process pool over one GPU: n shards, one stream (pool.hpp:47-94).
    Every op is one or more kernels per shard on the pool's stream."""

    def __init__(self, n: int, layout: ShardLayout, device: int = 0):
        validate_layout(layout)
        if n != layout.worker_count():
            raise LayoutError("worker count does not match layout shard count")
        self._layout = layout
        self.device = torch.device("cuda", device)

    def layout(self) -> ShardLayout:
        return self._layout

    def worker_count(self) -> int:
        return self._layout.worker_count()


def make_pool(dim: int, n: int) -> WorkerPool:
    return WorkerPool(min(n, dim), split_evenly(dim, n))


def make_sharded(layout: ShardLayout, prec: int, device=None) -> ShardedVector:
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return ShardedVector(layout, prec, [torch.zeros(e - b, dtype=_DTYPE[prec], device=dev)
                                        for b, e in layout.shard_bounds])


def _check_pool(pool: WorkerPool, a: ShardedVector):
    if a.layout != pool.layout():
        raise LayoutError("sharded vector does not belong to this pool's layout")


def _check_same(pool, a, b):
    _check_pool(pool, a)
    if a.layout != b.layout:
        raise LayoutError("sharded vectors have different layouts")
    if a.prec != b.prec:
        raise LayoutError("sharded vectors have different precision")


def _scalar(x: float, device) -> torch.Tensor:
    return torch.tensor([x], dtype=torch.float64, device=device)


def _fold(layout: ShardLayout, parts: list, m: int, device, post_sqrt=False) -> torch.Tensor:
    """Rank-ordered combine of per-shard partials (reduction.hpp:76-107), on device."""
    pstride = max(p.shape[-1] for p in parts)
    buf = torch.zeros(len(parts), m, pstride, dtype=torch.float64, device=device)
    for r, p in enumerate(parts):
        buf[r, :, :p.shape[-1]] = p.view(m, -1)
    out = torch.empty(m, dtype=torch.float64, device=device)
    n = layout.worker_count()
    ends = layout.ends
    plens = [lib().sd_partial_len(b, e, layout.total_dim) for b, e in layout.shard_bounds]
    if any(pl != pstride for pl in plens) and n > 1:
        pass  # the combine kernel reads each rank's own length inside the padded stride
    check(lib().sd_k_combine(n, _u64(layout.begins), _u64(ends), layout.total_dim, m, C.c_void_p(buf.data_ptr()),
                             C.c_void_p(out.data_ptr()), _stream()))
    return out.sqrt() if post_sqrt else out


def draw_probe(pool: WorkerPool, spec=None, prec: int = F64, *, seed=42, distribution=GAUSSIAN, one_hot_index=0,
               normalize=True) -> ShardedVector:
    """sharded.cpp:59-83."""
    if spec is not None:
        seed, distribution, one_hot_index, normalize = (spec.seed, spec.distribution, spec.one_hot_index,
                                                        spec.normalize)
    layout = pool.layout()
    if distribution == ONE_HOT and one_hot_index >= layout.total_dim:
        raise ArgumentError("one_hot index out of range")
    v = make_sharded(layout, prec, pool.device)
    for (b, e), t in zip(layout.shard_bounds, v.shards):
        check(lib().sd_k_probe_fill(C.c_void_p(t.data_ptr()), b, e, seed, distribution, one_hot_index, prec,
                                    _stream()))
    if normalize:
        n = norm2(pool, v)
        if not (n > 0.0):
            raise NumericalError("probe has zero norm")
        v = scale(pool, v, 1.0 / n)
    return v


@dataclass
class ProbeSpec:
    seed: int = 42
    distribution: int = GAUSSIAN
    one_hot_index: int = 0
    normalize: bool = True


def _dot_dev(pool, a: ShardedVector, b: ShardedVector) -> torch.Tensor:
    layout = a.layout
    parts = []
    for (s, e), ta, tb in zip(layout.shard_bounds, a.shards, b.shards):
        p = torch.empty(lib().sd_partial_len(s, e, layout.total_dim), dtype=torch.float64, device=ta.device)
        check(lib().sd_k_dot_partial(C.c_void_p(ta.data_ptr()), C.c_void_p(tb.data_ptr()), s, e, layout.total_dim,
                                     a.prec, C.c_void_p(p.data_ptr()), _stream()))
        parts.append(p)
    return _fold(layout, parts, 1, pool.device)


def dot(pool: WorkerPool, a: ShardedVector, b: ShardedVector) -> float:
    """sharded.cpp:85-100: ordered blocked f64 fold, bit-identical for every layout."""
    _check_same(pool, a, b)
    return float(_dot_dev(pool, a, b).item())


def norm2(pool: WorkerPool, x: ShardedVector) -> float:
    return math.sqrt(dot(pool, x, x))


def axpy(pool: WorkerPool, alpha: float, x: ShardedVector, y: ShardedVector) -> ShardedVector:
    """sharded.cpp:106-118: round(y + alpha*x) into a fresh vector."""
    _check_same(pool, x, y)
    out = ShardedVector(x.layout, x.prec, [t.clone() for t in y.shards])
    a = _scalar(alpha, pool.device)
    for tx, to in zip(x.shards, out.shards):
        check(lib().sd_k_axpy(C.c_void_p(tx.data_ptr()), C.c_void_p(to.data_ptr()), tx.numel(),
                              C.c_void_p(a.data_ptr()), 1.0, x.prec, _stream()))
    return out


def scale(pool: WorkerPool, x: ShardedVector, c: float) -> ShardedVector:
    """sharded.cpp:120-130."""
    if not math.isfinite(c):
        raise ArgumentError("scale factor is not finite")
    _check_pool(pool, x)
    out = make_sharded(x.layout, x.prec, pool.device)
    cc = _scalar(c, pool.device)
    for tx, to in zip(x.shards, out.shards):
        check(lib().sd_k_scale(C.c_void_p(tx.data_ptr()), C.c_void_p(to.data_ptr()), tx.numel(),
                               C.c_void_p(cc.data_ptr()), 0, x.prec, _stream()))
    return out


def gather(pool: WorkerPool, x: ShardedVector) -> np.ndarray:
    """sharded.cpp:132-140: full logical vector on the host (f64)."""
    _check_pool(pool, x)
    return torch.cat([t.double() for t in x.shards]).cpu().numpy()


def scatter(pool: WorkerPool, full, prec: int) -> ShardedVector:
    """sharded.cpp:142-154: distribute and round to prec."""
    layout = pool.layout()
    full = np.asarray(full, dtype=np.float64)
    if full.size != layout.total_dim:
        raise LayoutError("scatter source length does not match layout")
    dev = pool.device
    t = torch.from_numpy(full).to(dev)
    return ShardedVector(layout, prec, [t[b:e].to(_DTYPE[prec]).contiguous() for b, e in layout.shard_bounds])


# ---------------------------------------------------------------- operators
class OperatorHandle:
    """operators.hpp:15-21. apply() checks the dimension (layout_error) and
    returns a fresh vector; the native handle is what the Lanczos engine drives."""

    def __init__(self, dim: int, label: str, handle, keepalive=None):
        self.dim = dim
        self.label = label
        self._h = handle
        self._keep = keepalive

    @property
    def handle(self):
        return self._h

    def apply(self, pool: WorkerPool, x: ShardedVector) -> ShardedVector:
        if x.dim() != self.dim:
            raise LayoutError("operator/vector dimension mismatch")
        y = make_sharded(x.layout, x.prec, pool.device)
        full = torch.cat(x.shards) if len(x.shards) > 1 else x.shards[0]
        for (b, e), ty in zip(x.layout.shard_bounds, y.shards):
            if len(x.shards) == 1:
                check(lib().sd_operator_apply(self._h, C.c_void_p(full.data_ptr()), C.c_void_p(ty.data_ptr()),
                                              x.prec, _stream()))
            else:
                yf = torch.empty_like(full)
                check(lib().sd_operator_apply(self._h, C.c_void_p(full.data_ptr()), C.c_void_p(yf.data_ptr()),
                                              x.prec, _stream()))
                ty.copy_(yf[b:e])
        return y

    def __del__(self):
        try:
            if self._h:
                lib().sd_operator_destroy(self._h)
        except Exception:
            pass


DENSE_CAP = 2048


def dense_operator(a: np.ndarray, label: str = "dense") -> OperatorHandle:
    """operators.cpp:26-48."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    h = C.c_void_p()
    check(lib().sd_operator_dense(n, a.ctypes.data_as(_lib.dp), C.byref(h)))
    return OperatorHandle(n, label, h)


def wigner_dense(n: int, sigma: float, seed: int) -> np.ndarray:
    out = np.empty((n, n), np.float64)
    check(lib().sd_wigner_dense(n, sigma, seed, out.ctypes.data_as(_lib.dp)))
    return out


def spiked_dense(n: int, sigma: float, spikes, seed: int) -> np.ndarray:
    sp = np.ascontiguousarray(spikes, np.float64)
    out = np.empty((n, n), np.float64)
    check(lib().sd_spiked_dense(n, sigma, sp.ctypes.data_as(_lib.dp), sp.size, seed, out.ctypes.data_as(_lib.dp)))
    return out


def wigner_operator(n: int, sigma: float, seed: int) -> OperatorHandle:
    return dense_operator(wigner_dense(n, sigma, seed), f"wigner(n={n},sigma={sigma:g},seed={seed})")


def spiked_operator(n: int, sigma: float, spikes, seed: int) -> OperatorHandle:
    return dense_operator(spiked_dense(n, sigma, spikes, seed), f"spiked(n={n},seed={seed})")


def diag_operator(d: torch.Tensor, label: str = "diag") -> OperatorHandle:
    """Diagonal test operator y = round(d*x) on a device tensor (kept alive)."""
    prec = F32 if d.dtype == torch.float32 else F64
    h = C.c_void_p()
    check(lib().sd_operator_diag(d.numel(), C.c_void_p(d.data_ptr()), prec, C.byref(h)))
    return OperatorHandle(d.numel(), label, h, keepalive=d)


def custom_operator(dim: int, fn, label="custom") -> OperatorHandle:
    """fn(x_ptr, y_ptr, stream_ptr) -> None on raw device pointers."""
    def _cb(ctx, x, y, s):
        try:
            fn(x, y, s)
            return 0
        except Exception:  # surfaced as numerical_error by the engine
            return 4
    cb = _lib.APPLY_FN(_cb)
    h = C.c_void_p()
    check(lib().sd_operator_custom(dim, cb, None, C.byref(h)))
    return OperatorHandle(dim, label, h, keepalive=cb)


# ------------------------------------------------------------------ Lanczos
@dataclass
class LanczosConfig:
    """SPEC.md:241-243."""
    k_max: int = 10
    eps: float = -1.0
    reorthogonalize: int = REORTH_NONE
    probe: ProbeSpec = field(default_factory=ProbeSpec)
    prec: int = F64
    selective_window: int = 0  # REORTH_SELECTIVE: 2xCGS over the most recent W columns (ring of W)
    # REDUCE_ORDERED: the reference's 1024-block fold (bitwise parity mode);
    # REDUCE_TREE: fused GEMV passes with fixed-order tree reductions (HVP operators)
    reduction: int = 0

    def native(self) -> _lib.LanczosConfig:
        return _lib.LanczosConfig(self.k_max, self.eps, self.reorthogonalize, self.prec, self.probe.seed,
                                  self.probe.distribution, self.selective_window, self.reduction)


@dataclass
class LanczosResult:
    alphas: np.ndarray
    betas: np.ndarray
    breakdown: bool
    numerical_failure: bool
    ms_apply: float = 0.0
    ms_recurrence: float = 0.0
    ms_reorth: float = 0.0
    basis: np.ndarray | None = None


class Lanczos:
    """Step-level handle on the device engine (sd_lanczos_begin/step/end)."""

    def __init__(self, op: OperatorHandle, cfg: LanczosConfig, layout: ShardLayout | None = None, comm=None,
                 device=None, workspace: torch.Tensor | None = None):
        self.cfg = cfg
        self.total = op.dim
        self.layout = layout or ShardLayout(op.dim, ((0, op.dim),))
        n = self.layout.worker_count()
        self._b, self._e = _u64(self.layout.begins), _u64(self.layout.ends)
        self._cfg = cfg.native()
        self.comm = comm
        rank = comm.rank if comm is not None else 0
        nbytes = lib().sd_lanczos_workspace_bytes(self._b, self._e, op.dim, C.byref(self._cfg), n, rank)
        if nbytes == 0:
            check(1)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        if workspace is not None and workspace.numel() >= nbytes:
            self.workspace = workspace
        else:
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.op = op
        self.h = C.c_void_p()
        check(lib().sd_lanczos_begin(op.handle, comm.handle if comm is not None else None, self._b, self._e, op.dim,
                                     C.byref(self._cfg), C.c_void_p(self.workspace.data_ptr()), nbytes, _stream(),
                                     C.byref(self.h)))
        self.done = False

    def step(self) -> bool:
        d = C.c_int(0)
        check(lib().sd_lanczos_step(self.h, C.byref(d)))
        self.done = bool(d.value)
        return self.done

    def result(self, with_basis: bool = False) -> LanczosResult:
        k = self.cfg.k_max
        al = np.zeros(k, np.float64)
        be = np.zeros(k, np.float64)
        info = _lib.LanczosInfo()
        check(lib().sd_lanczos_result(self.h, al.ctypes.data_as(_lib.dp), be.ctypes.data_as(_lib.dp),
                                      C.byref(info)))
        res = LanczosResult(al[:info.n_alpha].copy(), be[:info.n_beta].copy(), bool(info.breakdown),
                            bool(info.numerical_failure), info.ms_apply, info.ms_recurrence, info.ms_reorth)
        if with_basis:
            ptr = C.c_void_p()
            nc = C.c_uint64()
            check(lib().sd_lanczos_basis(self.h, C.byref(ptr), C.byref(nc)))
            P = self.layout.shard_bounds[0][1] - self.layout.shard_bounds[0][0]
            ld = int(lib().sd_lanczos_basis_ld(self.h))
            off = (ptr.value - self.workspace.data_ptr())
            es = 4 if self.cfg.prec == F32 else 8
            Q = self.workspace[off:off + nc.value * ld * es].view(_DTYPE[self.cfg.prec]).view(nc.value, ld)[:, :P]
            res.basis = Q.double().cpu().numpy()
        return res

    def loss_of_orthogonality(self) -> float:
        """max_{i != j} |q_i^T q_j| over the stored basis
        (reference dots on the device); StateError without a stored basis."""
        out = C.c_double()
        check(lib().sd_lanczos_orthogonality(self.h, C.byref(out)))
        return out.value

    def close(self):
        if self.h:
            lib().sd_lanczos_end(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lanczos_run(op: OperatorHandle, cfg: LanczosConfig, with_basis: bool = False, layout=None,
                comm=None) -> LanczosResult:
    """SPEC.md:257-265. Raises NumericalError on non-finite alpha/beta (the
    partial tridiagonal rides on the exception as .result)."""
    if cfg.k_max < 1:
        raise ConfigError("k_max must be >= 1")
    L = Lanczos(op, cfg, layout, comm)
    try:
        while not L.step():
            pass
        res = L.result(with_basis=with_basis and cfg.reorthogonalize == REORTH_FULL)
    finally:
        L.close()
    if res.numerical_failure:
        e = NumericalError("non-finite alpha or beta")
        e.result = res
        raise e
    return res


# --------------------------------------------------------------- quadrature
@dataclass
class RitzSpectrum:
    values: np.ndarray
    weights: np.ndarray
    residual: float = 0.0


def ritz_decompose(alphas, betas) -> RitzSpectrum:
    """SPEC.md:319-327 (host, implicit-shift QL)."""
    al = np.ascontiguousarray(alphas, np.float64)
    be = np.ascontiguousarray(betas, np.float64)
    k = al.size
    if be.size != max(k - 1, 0):
        raise ArgumentError("tridiagonal needs k alphas and k-1 betas")
    v = np.empty(k, np.float64)
    w = np.empty(k, np.float64)
    r = C.c_double()
    check(lib().sd_ritz_decompose(k, al.ctypes.data_as(_lib.dp), be.ctypes.data_as(_lib.dp) if be.size else None,
                                  v.ctypes.data_as(_lib.dp), w.ctypes.data_as(_lib.dp), C.byref(r)))
    return RitzSpectrum(v, w, r.value)


@dataclass
class SmoothedDensity:
    grid: np.ndarray
    density: np.ndarray
    kernel_sigma: float


def smooth_density(s: RitzSpectrum, sigma: float = -1.0, grid_points: int = 512) -> SmoothedDensity:
    """SPEC.md:328-336."""
    k = s.values.size
    g = np.empty(grid_points, np.float64)
    d = np.empty(grid_points, np.float64)
    su = C.c_double()
    v = np.ascontiguousarray(s.values, np.float64)
    w = np.ascontiguousarray(s.weights, np.float64)
    check(lib().sd_smooth_density(k, v.ctypes.data_as(_lib.dp), w.ctypes.data_as(_lib.dp), sigma, grid_points,
                                  g.ctypes.data_as(_lib.dp), d.ctypes.data_as(_lib.dp), C.byref(su)))
    return SmoothedDensity(g, d, su.value)


def average_spectra(runs) -> RitzSpectrum:
    """union of (theta, w/n_runs), renormalised."""
    if not runs:
        raise ArgumentError("average_spectra needs at least one run")
    v = np.concatenate([r.values for r in runs])
    w = np.concatenate([r.weights for r in runs]) / len(runs)
    o = np.argsort(v, kind="stable")
    return RitzSpectrum(v[o], w[o] / w.sum())


# ------------------------------------------------------------- communication
class Comm:
    """An NCCL communicator owned by the C++ engine (one process per GPU).
    torch.distributed is only the bootstrap: it carries the ncclUniqueId."""

    def __init__(self, handle, rank: int, nranks: int):
        self.handle, self.rank, self.nranks = handle, rank, nranks

    def close(self):
        if self.handle:
            lib().sd_comm_destroy(self.handle)
            self.handle = None


def nccl_comm() -> Comm:
    import torch.distributed as dist
    rank, n = dist.get_rank(), dist.get_world_size()
    uid = C.create_string_buffer(128)
    if rank == 0:
        check(lib().sd_nccl_unique_id(uid))
    obj = [bytes(uid.raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    h = C.c_void_p()
    check(lib().sd_comm_nccl_create(C.create_string_buffer(obj[0], 128), n, rank, C.byref(h)))
    return Comm(h, rank, n)


def local_comms(n: int) -> list:
    """n in-process workers on the current device (the reference's WorkerPool
    model, pool.hpp:47-94): worker r's Comm, to be driven from its own thread
    with its own CUDA stream (see run_workers)."""
    arr = (C.c_void_p * n)()
    check(lib().sd_comm_local_create(n, arr))
    return [Comm(C.c_void_p(arr[r]), r, n) for r in range(n)]


def run_workers(n: int, fn):
    """Runs fn(rank, comm) on n worker threads of this process, each with its
    own CUDA stream on the current device; returns the results in rank order
    and re-raises the lowest-rank worker's exception (pool.cpp:54-64)."""
    import threading
    comms = local_comms(n)
    dev = torch.cuda.current_device()
    out, err = [None] * n, [None] * n

    def body(r):
        torch.cuda.set_device(dev)
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(r, comms[r])
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001 -- surfaced below in rank order
            err[r] = e
            lib().sd_comm_abort(comms[r].handle)  # release the workers waiting on this one
    ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for c in comms:
        c.close()
    # the lowest-rank ORIGINAL failure (pool.cpp:54-64); workers released by the
    # abort only report the abort
    real = [e for e in err if e is not None and not (isinstance(e, ProtocolError) and "aborted" in str(e))]
    for e in real or [e for e in err if e is not None]:
        raise e
    return out

