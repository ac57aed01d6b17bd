"""Stochastic Lanczos quadrature runs and their artifacts -- the consumer of
the hot path (SPEC.md quadrature :302-368 and the cmd_slq / compare_ortho
operations of the cli module :560-600, as library calls).

slq() runs the device Lanczos engine once per probe seed, decomposes every
tridiagonal (ritz_decompose), averages the spectra (average_spectra), smooths
the union (smooth_density) and, given an output directory, writes the
artifact files atomically (temp + rename) with round-trip float formatting so
identical runs produce byte-identical files (SPEC cli invariants)."""
from __future__ import annotations

import dataclasses
import os
import time

import numpy as np

from ._lib import ConfigError, NumericalError
from .core import (F32, REORTH_FULL, REORTH_NONE, DENSE_CAP, LanczosConfig, ProbeSpec, RitzSpectrum,
                   SmoothedDensity, average_spectra, lanczos_run, ritz_decompose, smooth_density)
from .diagnostics import GhostReport, PrecisionReport, detect_ghosts, precision_report

ARTIFACT_VERSION = 1


@dataclasses.dataclass
class ProbeRun:
    seed: int
    alphas: np.ndarray
    betas: np.ndarray
    spectrum: RitzSpectrum
    ghosts: GhostReport
    breakdown: bool
    seconds: float


@dataclasses.dataclass
class SlqArtifact:
    label: str
    config: LanczosConfig
    runs: list
    spectrum: RitzSpectrum
    density: SmoothedDensity
    ghosts: GhostReport
    precision: PrecisionReport
    files: dict = dataclasses.field(default_factory=dict)


def _f(x) -> str:
    return repr(float(x))


def _atomic_write(path: str, text: str) -> None:
    tmp = f"{path}.tmp.{os.getpid()}"
    with open(tmp, "w") as f:
        f.write(text)
    os.replace(tmp, path)


def spectrum_csv(s: RitzSpectrum) -> str:
    """(ritz_value, weight) -- the paper's Table layout (SPEC quadrature)."""
    return "ritz_value,weight\n" + "".join(f"{_f(v)},{_f(w)}\n" for v, w in zip(s.values, s.weights))


def density_csv(d: SmoothedDensity) -> str:
    return "x,density\n" + "".join(f"{_f(x)},{_f(y)}\n" for x, y in zip(d.grid, d.density))


def _report_text(a: SlqArtifact) -> str:
    c = a.config
    lines = [f"specden-b200 artifact v{ARTIFACT_VERSION}",
             f"operator = {a.label}",
             f"lanczos.k_max = {c.k_max}",
             f"lanczos.reorthogonalize = {'full' if c.reorthogonalize == REORTH_FULL else 'none'}",
             f"lanczos.precision = {'f32' if c.prec == F32 else 'f64'}",
             f"lanczos.breakdown_tol = {_f(c.eps)}",
             f"probe.distribution = {c.probe.distribution}",
             f"probe.seeds = {','.join(str(r.seed) for r in a.runs)}",
             f"precision.unit_roundoff = {_f(a.precision.unit_roundoff)}",
             f"precision.weight_rel_bound = {_f(a.precision.weight_rel_bound)}",
             f"ghosts.cluster_tol = {_f(a.ghosts.cluster_tol)}",
             f"ghosts.weight_threshold = {_f(a.ghosts.weight_threshold)}",
             f"ghosts.flagged_in_average = {a.ghosts.n_ghosts}"]
    for r in a.runs:
        lines.append(f"run.{r.seed}.k = {r.alphas.size}")
        lines.append(f"run.{r.seed}.breakdown = {int(r.breakdown)}")
        lines.append(f"run.{r.seed}.ghosts = {r.ghosts.n_ghosts}")
        lines.append(f"run.{r.seed}.alphas = {' '.join(_f(x) for x in r.alphas)}")
        lines.append(f"run.{r.seed}.betas = {' '.join(_f(x) for x in r.betas)}")
    return "\n".join(lines) + "\n"


def write_artifact(a: SlqArtifact, out_dir: str, timing: bool = False) -> dict:
    os.makedirs(out_dir, exist_ok=True)
    files = {"spectrum": os.path.join(out_dir, "spectrum.csv"), "density": os.path.join(out_dir, "density.csv"),
             "report": os.path.join(out_dir, "report.txt")}
    _atomic_write(files["spectrum"], spectrum_csv(a.spectrum))
    _atomic_write(files["density"], density_csv(a.density))
    _atomic_write(files["report"], _report_text(a))
    for r in a.runs:
        p = os.path.join(out_dir, f"spectrum_seed{r.seed}.csv")
        _atomic_write(p, spectrum_csv(r.spectrum))
        files[f"spectrum_seed{r.seed}"] = p
    if timing:  # wall times vary run to run: kept out of the byte-stable files
        p = os.path.join(out_dir, "timing.txt")
        _atomic_write(p, "".join(f"run.{r.seed}.seconds = {r.seconds:.6f}\n" for r in a.runs))
        files["timing"] = p
    a.files = files
    return files


def slq(op, cfg: LanczosConfig, seeds, out_dir: str | None = None, sigma: float = -1.0, grid_points: int = 512,
        cluster_tol: float = 1e-6, weight_threshold: float = 1e-8, layout=None, comm=None,
        label: str | None = None) -> SlqArtifact:
    """cmd_slq: one Lanczos run per probe seed, averaged spectrum, density,
    ghost and precision reports. A numerical breakdown (non-finite alpha or
    beta) still writes the partial artifact before re-raising."""
    seeds = [int(s) for s in seeds]
    if not seeds:
        raise ConfigError("slq needs at least one probe seed")
    runs, failure = [], None
    for sd_ in seeds:
        c = dataclasses.replace(cfg, probe=dataclasses.replace(cfg.probe, seed=sd_))
        t0 = time.perf_counter()
        try:
            res = lanczos_run(op, c, layout=layout, comm=comm)
        except NumericalError as e:
            res, failure = getattr(e, "result", None), e
            if res is None or res.alphas.size == 0:
                raise
        spec = ritz_decompose(res.alphas, res.betas)
        runs.append(ProbeRun(sd_, res.alphas, res.betas, spec, detect_ghosts(spec, cluster_tol, weight_threshold),
                             bool(res.breakdown), time.perf_counter() - t0))
        if failure:
            break
    avg = average_spectra([r.spectrum for r in runs])
    art = SlqArtifact(label or getattr(op, "label", "operator"), cfg, runs, avg,
                      smooth_density(avg, sigma, grid_points), detect_ghosts(avg, cluster_tol, weight_threshold),
                      precision_report(cfg.prec, max(r.alphas.size for r in runs)))
    if out_dir is not None:
        write_artifact(art, out_dir)
    if failure:
        failure.artifact = art
        raise failure
    return art


@dataclasses.dataclass
class CompareOrtho:
    none: SlqArtifact
    full: SlqArtifact

    def table(self) -> str:
        """Side-by-side Ritz tables with ghost flags (SPEC cmd_compare_ortho)."""
        a, b = self.none, self.full
        k = max(a.spectrum.values.size, b.spectrum.values.size)
        rows = ["no_ortho_value,no_ortho_weight,no_ortho_ghost,full_ortho_value,full_ortho_weight,full_ortho_ghost"]
        for i in range(k):
            cells = []
            for art in (a, b):
                if i < art.spectrum.values.size:
                    cells += [_f(art.spectrum.values[i]), _f(art.spectrum.weights[i]),
                              str(int(art.ghosts.ghost_flags[i]))]
                else:
                    cells += ["", "", ""]
            rows.append(",".join(cells))
        return "\n".join(rows) + "\n"


def compare_ortho(op, cfg: LanczosConfig, seed: int, out_dir: str | None = None, **kw) -> CompareOrtho:
    """Run no-ortho and full-ortho with the identical probe (Fig. 3 c/d)."""
    a = slq(op, dataclasses.replace(cfg, reorthogonalize=REORTH_NONE), [seed], **kw)
    b = slq(op, dataclasses.replace(cfg, reorthogonalize=REORTH_FULL), [seed], **kw)
    out = CompareOrtho(a, b)
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        write_artifact(a, os.path.join(out_dir, "no_ortho"))
        write_artifact(b, os.path.join(out_dir, "full_ortho"))
        _atomic_write(os.path.join(out_dir, "compare.csv"), out.table())
    return out


def load_dense(path: str) -> np.ndarray:
    """Dense operator file (load_dense, proj/src/operators.cpp:114-135):
    header 'dim N', then N*N whitespace-separated reals; symmetry validated."""
    try:
        text = open(path).read()
    except OSError:
        raise ConfigError(f"cannot open dense operator file '{path}'") from None
    tok = text.split()
    if len(tok) < 2 or tok[0] != "dim":
        raise ConfigError("dense operator file must start with a 'dim N' header")
    try:
        n = int(tok[1])
    except ValueError:
        raise ConfigError("dense operator file must start with a 'dim N' header") from None
    if n < 2 or n > DENSE_CAP:
        from ._lib import ArgumentError
        raise ArgumentError("dense operators need n >= 2" if n < 2 else
                            f"dense operator size exceeds the desk-scale cap ({DENSE_CAP})")
    vals = tok[2:]
    if len(vals) < n * n:
        raise ConfigError(f"dense operator file ended early (expected {n}x{n} entries)")
    try:
        a = np.array([float(x) for x in vals[:n * n]], np.float64).reshape(n, n)
    except ValueError:
        raise ConfigError(f"dense operator file ended early (expected {n}x{n} entries)") from None
    for i in range(n):
        for j in range(i + 1, n):
            if a[i, j] != a[j, i]:
                raise ConfigError(f"dense operator file is not symmetric at ({i},{j})")
    return a


__all__ = ["slq", "compare_ortho", "load_dense", "write_artifact", "spectrum_csv", "density_csv", "SlqArtifact",
           "ProbeRun", "CompareOrtho", "ProbeSpec"]
