"""Hessian-column probing (SPEC.md column_probe module; §Banded
Hessians): one-hot operator applies, and the 50-bin |x| histogram plus the
strict threshold-fraction table 1e-12 ... 1e-1 of a column, computed on the
device in two HBM passes (sd_k_abs_stats, sd_k_abs_histogram)."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from ._lib import ArgumentError, check, lib
from .core import ONE_HOT, ShardedVector, WorkerPool, _stream, draw_probe

THRESHOLDS = tuple(float(f"1e-{k}") for k in range(12, 0, -1))  # 1e-12 .. 1e-1 (SPEC default grid)


@dataclass
class ColumnProbeReport:
    column_index: int
    bin_edges: np.ndarray          # bins + 1 edges over [0, max|x|]
    counts: np.ndarray             # bins
    thresholds: tuple
    fractions: np.ndarray          # fraction of entries with |x| < t (strict)
    total_elements: int
    seed: int | None = None
    max_abs: float = 0.0
    below: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


def probe_column(op, pool: WorkerPool, index: int, prec: int) -> ShardedVector:
    """SPEC probe_column: op applied to e_index (the index-th column)."""
    if not (0 <= index < op.dim):
        raise ArgumentError("column index out of range")
    e = draw_probe(pool, None, prec, seed=0, distribution=ONE_HOT, one_hot_index=index, normalize=False)
    return op.apply(pool, e)


def column_report(col: ShardedVector, index: int, thresholds=THRESHOLDS, bins: int = 50,
                  seed: int | None = None) -> ColumnProbeReport:
    """SPEC column_report: per-shard device statistics, combined exactly
    (max of maxima, integer sums) -> shard-layout invariant."""
    thr = np.ascontiguousarray(thresholds, np.float64)
    below = np.zeros(thr.size, np.uint64)
    mx = 0.0
    n_total = 0
    for t in col.shards:
        c = np.zeros(thr.size, np.uint64)
        m = C.c_double()
        check(lib().sd_k_abs_stats(C.c_void_p(t.data_ptr()), t.numel(), col.prec, thr.ctypes.data, int(thr.size),
                                   c.ctypes.data, C.byref(m), _stream()))
        below += c
        mx = max(mx, m.value)
        n_total += t.numel()
    counts = np.zeros(bins, np.uint64)
    for t in col.shards:
        c = np.zeros(bins, np.uint64)
        check(lib().sd_k_abs_histogram(C.c_void_p(t.data_ptr()), t.numel(), col.prec, mx, bins, c.ctypes.data,
                                       _stream()))
        counts += c
    edges = np.linspace(0.0, mx, bins + 1) if mx > 0 else np.zeros(bins + 1)
    return ColumnProbeReport(index, edges, counts, tuple(float(x) for x in thr), below / float(n_total), n_total,
                             seed, mx, below)


def multi_seed_probe(op, pool: WorkerPool, seeds, prec: int, thresholds=THRESHOLDS, bins: int = 50):
    """SPEC multi_seed_probe: column index uniform_index(seed, 0, P) per seed
    (rng.hpp:50-52), one report per seed."""
    reports = []
    for s in seeds:
        idx = int(lib().sd_uniform_index(int(s), 0, op.dim))
        col = probe_column(op, pool, idx, prec)
        reports.append(column_report(col, idx, thresholds, bins, seed=int(s)))
    return reports


def _atomic_write(path: str, text: str) -> None:
    tmp = f"{path}.tmp.{os.getpid()}"
    with open(tmp, "w") as f:
        f.write(text)
    os.replace(tmp, path)


def write_report(report: ColumnProbeReport, out_dir: str, stem: str | None = None) -> tuple[str, str]:
    """CSV exports (SPEC column_probe External Interfaces): (threshold,
    fraction) and (bin_left, bin_right, count); full round-trip formatting."""
    os.makedirs(out_dir, exist_ok=True)
    stem = stem or f"column_{report.column_index}" + (f"_seed{report.seed}" if report.seed is not None else "")
    fr = "threshold,fraction\n" + "".join(
        f"{float(t)!r},{float(f)!r}\n" for t, f in zip(report.thresholds, report.fractions))
    hi = "bin_left,bin_right,count\n" + "".join(
        f"{float(report.bin_edges[i])!r},{float(report.bin_edges[i + 1])!r},{int(report.counts[i])}\n"
        for i in range(report.counts.size))
    a, b = os.path.join(out_dir, stem + "_fractions.csv"), os.path.join(out_dir, stem + "_histogram.csv")
    _atomic_write(a, fr)
    _atomic_write(b, hi)
    return a, b
