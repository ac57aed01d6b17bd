"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the CPU restatement (oracle/liboracle.so, sources in
oracle/src) and for the compiled reference (oracle/_ref/libspecden_ref.so,
built in place from /root/reference/proj by oracle/build_ref.sh).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module; the product package
(paper_2505_11564_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libspecden_ref.so"

F32, F64 = 0, 1
GAUSSIAN, RADEMACHER, ONE_HOT = 0, 1, 2
ERR_NAMES = {1: "config_error", 2: "layout_error", 3: "argument_error", 4: "numerical_error",
             5: "state_error", 6: "protocol_error", 99: "error"}

_d = C.c_double
_dp = C.POINTER(C.c_double)
_ll = C.c_longlong
_llp = C.POINTER(C.c_longlong)
_ull = C.c_ulonglong
_up = C.POINTER(C.c_uint)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, "error")


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref/ when /root/reference exists)."""
    if force or not LIB.exists() or any(p.stat().st_mtime > LIB.stat().st_mtime for p in (HERE / "src").glob("*")):
        subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    if (force or not REF_LIB.exists()) and Path("/root/reference/proj/src").is_dir():
        subprocess.run([str(HERE / "build_ref.sh")], check=True, stdout=subprocess.DEVNULL)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _pl(a: np.ndarray):
    return a.ctypes.data_as(_llp)


def _pu(a: np.ndarray):
    return a.ctypes.data_as(_up)


class Oracle:
    def __init__(self, path: Path = LIB):
        if not path.exists():
            build()
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.oracle_last_error.restype = C.c_char_p
        for name, res, args in [
            ("oracle_mix64", _ull, [_ull]),
            ("oracle_keyed_counter", _ull, [_ull, _ull]),
            ("oracle_uniform01", _d, [_ull, _ull]),
            ("oracle_gaussian", _d, [_ull, _ull]),
            ("oracle_rademacher", _d, [_ull, _ull]),
            ("oracle_uniform_index", _ull, [_ull, _ull, _ull]),
            ("oracle_gaussian_fill", None, [_ull, _ull, _ll, _dp]),
            ("oracle_dot", _d, [_ll, _dp, _dp]),
            ("oracle_blocked_sum", _d, [_ll, _dp]),
            ("oracle_gpt_param_count", _ll, [_llp]),
            ("oracle_mlp_param_count", _ll, [_llp, _ll]),
        ]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    def _chk(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(rc, self.lib.oracle_last_error().decode())

    # ---- RNG
    def keyed_counter(self, s, c):
        return self.lib.oracle_keyed_counter(s, c)

    def mix64(self, x):
        return self.lib.oracle_mix64(x)

    def gaussian(self, s, i):
        return self.lib.oracle_gaussian(s, i)

    def rademacher(self, s, i):
        return self.lib.oracle_rademacher(s, i)

    def uniform01(self, s, i):
        return self.lib.oracle_uniform01(s, i)

    def uniform_index(self, s, i, n):
        return self.lib.oracle_uniform_index(s, i, n)

    def gaussian_fill(self, seed: int, first: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.oracle_gaussian_fill(seed, first, n, _p(out))
        return out

    # ---- layout / reduction / vectors
    def split_evenly(self, dim: int, n: int):
        b = np.zeros(max(n, 1), np.int64)
        e = np.zeros(max(n, 1), np.int64)
        cnt = np.zeros(1, np.int64)
        self._chk(self.lib.oracle_split_evenly(_ll(dim), _ll(n), _pl(b), _pl(e), _pl(cnt)))
        return [(int(b[i]), int(e[i])) for i in range(int(cnt[0]))]

    def validate_layout(self, total: int, ranges):
        b = np.array([r[0] for r in ranges], np.int64)
        e = np.array([r[1] for r in ranges], np.int64)
        self._chk(self.lib.oracle_validate_layout(_ll(total), _ll(len(ranges)), _pl(b), _pl(e)))

    def draw_probe(self, dim, seed=42, dist=GAUSSIAN, one_hot=0, normalize=True, prec=F64) -> np.ndarray:
        out = np.empty(dim, np.float64)
        self._chk(self.lib.oracle_draw_probe(_ll(dim), _ull(seed), dist, _ll(one_hot), int(normalize), prec, _p(out)))
        return out

    def dot(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self.lib.oracle_dot(a.size, _p(a), _p(b))

    def blocked_sum(self, terms: np.ndarray) -> float:
        t = np.ascontiguousarray(terms, np.float64)
        return self.lib.oracle_blocked_sum(t.size, _p(t))

    def axpy(self, alpha, x, y, prec=F64):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty_like(x)
        self._chk(self.lib.oracle_axpy(_ll(x.size), _d(alpha), _p(x), _p(y), prec, _p(out)))
        return out

    def scale(self, x, c, prec=F64):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self._chk(self.lib.oracle_scale(_ll(x.size), _p(x), _d(c), prec, _p(out)))
        return out

    def dot_partial(self, begin, end, total, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        buf = np.empty(end - begin + 2, np.float64)
        cnt = np.zeros(3, np.int64)
        self._chk(self.lib.oracle_dot_partial(_ll(begin), _ll(end), _ll(total), _p(a), _p(b), _p(buf), _pl(cnt)))
        h, s, t = (int(x) for x in cnt)
        return buf[:h].copy(), buf[h:h + s].copy(), buf[h + s:h + s + t].copy()

    def combine_partials(self, total, ranges, parts):
        b = np.array([r[0] for r in ranges], np.int64)
        e = np.array([r[1] for r in ranges], np.int64)
        cnt = np.array([len(x) for p in parts for x in p], np.int64)
        buf = np.concatenate([np.concatenate(p) for p in parts]).astype(np.float64)
        out = np.zeros(1, np.float64)
        self._chk(self.lib.oracle_combine_partials(_ll(len(ranges)), _ll(total), _pl(b), _pl(e), _pl(cnt),
                                                   _p(buf), _p(out)))
        return float(out[0])

    # ---- dense operators / Lanczos / quadrature
    def wigner(self, n, sigma, seed):
        out = np.empty((n, n), np.float64)
        self._chk(self.lib.oracle_wigner(_ll(n), _d(sigma), _ull(seed), _p(out)))
        return out

    def spiked(self, n, sigma, spikes, seed):
        sp = np.ascontiguousarray(spikes, np.float64)
        out = np.empty((n, n), np.float64)
        self._chk(self.lib.oracle_spiked(_ll(n), _d(sigma), _p(sp), _ll(sp.size), _ull(seed), _p(out)))
        return out

    def dense_apply(self, a, x, prec=F64):
        a = np.ascontiguousarray(a, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self._chk(self.lib.oracle_dense_apply(_ll(x.size), _p(a), _p(x), prec, _p(out)))
        return out

    def lanczos_dense(self, a, k_max, eps=-1.0, reorth=False, seed=42, dist=GAUSSIAN, prec=F64, basis=False, window=0):
        a = np.ascontiguousarray(a, np.float64)
        n = a.shape[0]
        al = np.zeros(k_max, np.float64)
        be = np.zeros(k_max, np.float64)
        sb = np.zeros(k_max, np.float64)
        info = np.zeros(5, np.int64)
        Q = np.zeros((k_max + 1, n), np.float64) if basis else None
        self._chk(self.lib.oracle_lanczos_dense(_ll(n), _p(a), _ll(k_max), _d(eps), int(reorth), _ll(window), _ull(seed), dist,
                                                prec, _p(al), _p(be), _p(sb), _p(Q) if basis else None, _pl(info)))
        res = {"alphas": al[:info[0]].copy(), "betas": be[:info[1]].copy(), "step_beta": sb[:info[0]].copy(),
               "breakdown": bool(info[2]), "numerical_failure": bool(info[3])}
        if basis:
            res["basis"] = Q[:info[4]].copy()
        return res

    def lanczos_diag(self, d, k_max, eps=-1.0, reorth=False, seed=42, dist=RADEMACHER, prec=F32, window=0):
        d = np.ascontiguousarray(d, np.float64)
        al = np.zeros(k_max, np.float64)
        be = np.zeros(k_max, np.float64)
        info = np.zeros(4, np.int64)
        self._chk(self.lib.oracle_lanczos_diag(_ll(d.size), _p(d), _ll(k_max), _d(eps), int(reorth), _ll(window), _ull(seed),
                                               dist,
                                               prec, _p(al), _p(be), _pl(info)))
        return {"alphas": al[:info[0]].copy(), "betas": be[:info[1]].copy(), "breakdown": bool(info[2])}

    def lanczos_gpt(self, cfg, theta, tok, tgt, B, S, k_max, eps=-1.0, reorth=True, seed=42, dist=RADEMACHER,
                    prec=F32, hvp_prec=F64, window=0):
        """Lanczos (oracle restatement of SPEC.md:257-265) over the oracle's own
        GPT HVP: the CPU leg of the C1 SLQ parity check."""
        c = self._cfg(cfg)
        th = np.ascontiguousarray(theta, np.float64)
        tok = np.ascontiguousarray(tok, np.uint32)
        tgt = np.ascontiguousarray(tgt, np.uint32)
        al = np.zeros(k_max, np.float64)
        be = np.zeros(k_max, np.float64)
        info = np.zeros(4, np.int64)
        self._chk(self.lib.oracle_lanczos_gpt(_pl(c), _p(th), _ll(B), _ll(S), _pu(tok), _pu(tgt), _ll(k_max), _d(eps),
                                              int(reorth), _ll(window), _ull(seed), dist, prec, hvp_prec, _p(al),
                                              _p(be), _pl(info)))
        return {"alphas": al[:info[0]].copy(), "betas": be[:info[1]].copy(), "breakdown": bool(info[2]),
                "numerical_failure": bool(info[3])}

    def ritz(self, alphas, betas):
        al = np.ascontiguousarray(alphas, np.float64)
        be = np.ascontiguousarray(betas, np.float64)
        k = al.size
        v = np.empty(k, np.float64)
        w = np.empty(k, np.float64)
        self._chk(self.lib.oracle_ritz(_ll(k), _p(al), _p(be) if be.size else None, _p(v), _p(w)))
        return v, w

    def smooth_density(self, values, weights, sigma=-1.0, npts=512):
        v = np.ascontiguousarray(values, np.float64)
        w = np.ascontiguousarray(weights, np.float64)
        g = np.empty(npts, np.float64)
        d = np.empty(npts, np.float64)
        s = np.zeros(1, np.float64)
        self._chk(self.lib.oracle_smooth_density(_ll(v.size), _p(v), _p(w), _d(sigma), _ll(npts), _p(g), _p(d),
                                                 _p(s)))
        return g, d, float(s[0])

    # ---- GPT / MLP autodiff
    @staticmethod
    def _cfg(cfg) -> np.ndarray:
        return np.array([cfg["n_layer"], cfg["d"], cfg["n_head"], cfg["ff"], cfg["vocab"], cfg["ctx"],
                         cfg.get("arch", 0), cfg.get("rope_base", 10000), cfg.get("n_kv_head", 0)], np.int64)

    def gpt_param_count(self, cfg) -> int:
        c = self._cfg(cfg)
        return self.lib.oracle_gpt_param_count(_pl(c))

    def gpt_layout(self, cfg):
        c = self._cfg(cfg)
        n = (4 + 12 * cfg["n_layer"]) if cfg.get("arch", 0) == 0 else (3 + 6 * cfg["n_layer"])
        off = np.zeros(n, np.int64)
        r = np.zeros(n, np.int64)
        co = np.zeros(n, np.int64)
        k = np.zeros(n, np.int32)
        cnt = np.zeros(1, np.int64)
        self._chk(self.lib.oracle_gpt_layout(_pl(c), _pl(off), _pl(r), _pl(co), k.ctypes.data_as(C.POINTER(C.c_int)),
                                             _pl(cnt)))
        return [(int(off[i]), int(r[i]), int(co[i]), int(k[i])) for i in range(int(cnt[0]))]

    def gpt_init(self, cfg, seed=0, gain_scale=0.0, bias_scale=0.0, prec=F64):
        c = self._cfg(cfg)
        out = np.empty(self.gpt_param_count(cfg), np.float64)
        self._chk(self.lib.oracle_gpt_init(_pl(c), _ull(seed), _d(gain_scale), _d(bias_scale), prec, _p(out)))
        return out

    def gpt_batch(self, cfg, B, S, seed_tok=1, first_seq=0):
        c = self._cfg(cfg)
        tok = np.empty(B * S, np.uint32)
        tgt = np.empty(B * S, np.uint32)
        self._chk(self.lib.oracle_gpt_batch(_pl(c), _ll(B), _ll(S), _ull(seed_tok), _ll(first_seq), _pu(tok), _pu(tgt)))
        return tok, tgt

    def gpt_loss(self, cfg, theta, tok, tgt, B, S, prec=F64):
        c = self._cfg(cfg)
        th = np.ascontiguousarray(theta, np.float64)
        out = np.zeros(1, np.float64)
        self._chk(self.lib.oracle_gpt_loss(_pl(c), _p(th), _ll(B), _ll(S), _pu(tok), _pu(tgt), prec, _p(out)))
        return float(out[0])

    def gpt_grad(self, cfg, theta, tok, tgt, B, S, prec=F64):
        c = self._cfg(cfg)
        th = np.ascontiguousarray(theta, np.float64)
        out = np.empty_like(th)
        self._chk(self.lib.oracle_gpt_grad(_pl(c), _p(th), _ll(B), _ll(S), _pu(tok), _pu(tgt), prec, _p(out)))
        return out

    def gpt_hvp(self, cfg, theta, tok, tgt, B, S, v, prec=F64):
        c = self._cfg(cfg)
        th = np.ascontiguousarray(theta, np.float64)
        vv = np.ascontiguousarray(v, np.float64)
        out = np.empty_like(th)
        self._chk(self.lib.oracle_gpt_hvp(_pl(c), _p(th), _ll(B), _ll(S), _pu(tok), _pu(tgt), _p(vv), prec, _p(out)))
        return out

    def gpt_batched_hvp(self, cfg, theta, batches, S, v, prec=F64):
        """batches: list of (B_i, tok_i, tgt_i)."""
        c = self._cfg(cfg)
        th = np.ascontiguousarray(theta, np.float64)
        vv = np.ascontiguousarray(v, np.float64)
        Bs = np.array([b[0] for b in batches], np.int64)
        tok = np.concatenate([b[1] for b in batches]).astype(np.uint32)
        tgt = np.concatenate([b[2] for b in batches]).astype(np.uint32)
        out = np.empty_like(th)
        self._chk(self.lib.oracle_gpt_batched_hvp(_pl(c), _p(th), _ll(len(batches)), _pl(Bs), _ll(S), _pu(tok),
                                                  _pu(tgt), _p(vv), prec, _p(out)))
        return out

    def mlp_param_count(self, widths):
        w = np.array(widths, np.int64)
        return self.lib.oracle_mlp_param_count(_pl(w), _ll(w.size))

    def mlp_grad(self, widths, theta, x, y, prec=F64):
        w = np.array(widths, np.int64)
        th = np.ascontiguousarray(theta, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty_like(th)
        self._chk(self.lib.oracle_mlp_grad(_pl(w), _ll(w.size), _p(th), _ll(x.shape[0]), _p(x), _p(y), prec, _p(out)))
        return out

    def mlp_hvp(self, widths, theta, x, y, v, prec=F64):
        w = np.array(widths, np.int64)
        th = np.ascontiguousarray(theta, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        vv = np.ascontiguousarray(v, np.float64)
        out = np.empty_like(th)
        self._chk(self.lib.oracle_mlp_hvp(_pl(w), _ll(w.size), _p(th), _ll(x.shape[0]), _p(x), _p(y), _p(vv), prec,
                                          _p(out)))
        return out


class Reference:
    """The compiled reference (oracle/_ref/libspecden_ref.so)."""

    def __init__(self, path: Path = REF_LIB):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (oracle/build_ref.sh needs /root/reference)")
        self.lib = C.CDLL(str(path))
        self.lib.refc_last_error.restype = C.c_char_p

    @staticmethod
    def available() -> bool:
        return REF_LIB.exists()

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.refc_last_error().decode())

    def draw_probe(self, dim, workers=1, seed=42, dist=GAUSSIAN, one_hot=0, normalize=True, prec=F64):
        out = np.empty(dim, np.float64)
        self._chk(self.lib.refc_draw_probe(_ll(dim), _ll(workers), _ull(seed), dist, _ll(one_hot), int(normalize),
                                           prec, _p(out)))
        return out

    def dot(self, a, b, workers=1, prec=F64):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros(1, np.float64)
        self._chk(self.lib.refc_dot(_ll(a.size), _ll(workers), _p(a), _p(b), prec, _p(out)))
        return float(out[0])

    def axpy(self, alpha, x, y, workers=1, prec=F64):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty_like(x)
        self._chk(self.lib.refc_axpy(_ll(x.size), _ll(workers), _d(alpha), _p(x), _p(y), prec, _p(out)))
        return out

    def scale(self, x, c, workers=1, prec=F64):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self._chk(self.lib.refc_scale(_ll(x.size), _ll(workers), _p(x), _d(c), prec, _p(out)))
        return out

    def wigner(self, n, sigma, seed):
        out = np.empty((n, n), np.float64)
        self._chk(self.lib.refc_wigner(_ll(n), _d(sigma), _ull(seed), _p(out)))
        return out

    def spiked(self, n, sigma, spikes, seed):
        sp = np.ascontiguousarray(spikes, np.float64)
        out = np.empty((n, n), np.float64)
        self._chk(self.lib.refc_spiked(_ll(n), _d(sigma), _p(sp), _ll(sp.size), _ull(seed), _p(out)))
        return out

    def dense_apply(self, a, x, workers=1, prec=F64):
        a = np.ascontiguousarray(a, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self._chk(self.lib.refc_dense_apply(_ll(x.size), _p(a), _ll(workers), _p(x), prec, _p(out)))
        return out

    def lanczos_dense(self, a, k_max, workers=1, eps=-1.0, reorth=False, seed=42, dist=GAUSSIAN, prec=F64):
        a = np.ascontiguousarray(a, np.float64)
        al = np.zeros(k_max, np.float64)
        be = np.zeros(k_max, np.float64)
        info = np.zeros(3, np.int64)
        self._chk(self.lib.refc_lanczos_dense(_ll(a.shape[0]), _p(a), _ll(workers), _ll(k_max), _d(eps), int(reorth),
                                              _ull(seed), dist, prec, _p(al), _p(be), _pl(info)))
        return {"alphas": al[:info[0]].copy(), "betas": be[:info[1]].copy(), "breakdown": bool(info[2])}

    def time_recurrence(self, dim, workers, j, reps=1, prec=F32) -> float:
        s = np.zeros(1, np.float64)
        self._chk(self.lib.refc_time_recurrence(_ll(dim), _ll(workers), _ll(j), _ll(reps), prec, _p(s)))
        return float(s[0])


_ORACLE = None


def oracle() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = Oracle()
    return _ORACLE


def nthreads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


def column_report(x, thresholds, bins=50):
    """CPU restatement of SPEC.md column_probe.column_report (strict |x| < t
    fractions; `bins` uniform bins over [0, max|x|], bin = min(bins-1,
    floor(|x| / max * bins)) in f64, all in bin 0 for an all-zero column).
    Test infrastructure only: the checker for sd_k_abs_stats/_histogram."""
    a = np.abs(np.asarray(x, np.float64))
    thr = np.asarray(thresholds, np.float64)
    below = np.array([(a < t).sum() for t in thr], np.uint64)
    mx = float(a.max()) if a.size else 0.0
    if mx > 0:
        b = np.minimum(np.floor(a / mx * float(bins)), bins - 1).astype(np.int64)
    else:
        b = np.zeros(a.size, np.int64)
    counts = np.bincount(b, minlength=bins).astype(np.uint64)
    return below, counts, mx
