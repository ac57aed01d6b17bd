"""Run diagnostics (SPEC.md diagnostics module, :370-434): ghost detection,
the floating-point weight-error bound, and near-zero (rank-degeneracy)
classification of Ritz pairs. Pure host functions on RitzSpectrum; they
annotate spectra and never mutate them (SPEC design decision)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import ArgumentError
from .core import F32, F64, RitzSpectrum


@dataclass
class GhostCluster:
    representative: float
    members: list
    total_weight: float


@dataclass
class GhostReport:
    clusters: list
    ghost_flags: np.ndarray
    cluster_tol: float
    weight_threshold: float

    @property
    def n_ghosts(self) -> int:
        return int(self.ghost_flags.sum())


def detect_ghosts(s: RitzSpectrum, cluster_tol: float = 1e-6, weight_threshold: float = 1e-8) -> GhostReport:
    """Single-linkage clusters of the ascending Ritz values with gaps <=
    cluster_tol * spectral width; inside a multi-member cluster every member
    but the heaviest whose weight is below weight_threshold * max weight is
    flagged (defaults: SPEC diagnostics design decisions)."""
    v = np.asarray(s.values, np.float64)
    w = np.asarray(s.weights, np.float64)
    k = v.size
    flags = np.zeros(k, bool)
    if k == 0:
        return GhostReport([], flags, cluster_tol, weight_threshold)
    order = np.argsort(v, kind="stable")
    width = float(v.max() - v.min())
    gap = cluster_tol * width
    wmax = float(w.max())
    clusters, cur = [], [order[0]]
    for a, b in zip(order[:-1], order[1:]):
        if v[b] - v[a] <= gap:
            cur.append(b)
        else:
            clusters.append(cur)
            cur = [b]
    clusters.append(cur)
    out = []
    for c in clusters:
        heavy = max(c, key=lambda i: (w[i], -i))
        if len(c) > 1:
            for i in c:
                if i != heavy and w[i] < weight_threshold * wmax:
                    flags[i] = True
        out.append(GhostCluster(float(v[heavy]), [float(v[i]) for i in c], float(w[c].sum())))
    return GhostReport(out, flags, cluster_tol, weight_threshold)


@dataclass
class PrecisionReport:
    unit_roundoff: float
    k: int
    weight_rel_bound: float
    machine_eps_threshold: float


def precision_report(prec: int, k: int) -> PrecisionReport:
    """|w_hat - w| / w <= 2 k u (PAPER §precision); machine epsilon 2^-23 in
    f32 (PAPER §rank degeneracy)."""
    if k < 1:
        raise ArgumentError("precision_report needs k >= 1")
    if prec == F32:
        u, eps = 2.0 ** -24, 2.0 ** -23
    elif prec == F64:
        u, eps = 2.0 ** -53, 2.0 ** -52
    else:
        raise ArgumentError("precision must be f32 or f64")
    return PrecisionReport(u, int(k), 2.0 * k * u, eps)


@dataclass
class NearZeroReport:
    near_zero_mass: float
    outlier_mass: float
    near_zero: np.ndarray  # boolean per Ritz pair


def classify_near_zero(s: RitzSpectrum, eps_threshold: float = 2.0 ** -23) -> NearZeroReport:
    """Ritz pairs with |theta| <= eps_threshold * spectral width are near
    zero (PAPER §rank degeneracy); both masses sum to the total weight."""
    v = np.asarray(s.values, np.float64)
    w = np.asarray(s.weights, np.float64)
    if v.size == 0:
        raise ArgumentError("empty spectrum")
    width = float(v.max() - v.min())
    nz = np.abs(v) <= eps_threshold * width
    tot = float(w.sum())
    a = float(w[nz].sum()) / tot
    return NearZeroReport(a, float(w[~nz].sum()) / tot, nz)
