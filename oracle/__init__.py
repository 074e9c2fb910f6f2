"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/cfust_oracle.c`` (plain FP64 CPU FM-CFUST EM written from
arXiv 2005.06848 and the DESIGN.md readings).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this package.  It
shares no code with ``paper_2005_06848_b200`` and never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cfust_oracle.c")
_LIB = os.path.join(_HERE, "libcfust_oracle.so")

OK, EINVAL, ENOTPD, EUNDERFLOW, EEMPTY = 0, -1, -4, -5, -6
E1_EXACT, FAMILY_SN, DIRECT = 1, 2, 4   # E-step / fit flags (reading R2'; family F1; SOV-direct D1)
FAMILIES = {"st": 0, "sn": FAMILY_SN}   # CFUST (skew-t, default) / CFUSN (skew-normal, nu = inf)


ESTIMATORS = {"analytic": 0, "direct": DIRECT}   # truncated moments: O6-O7 (default) / SOV-direct (D1)


def _flags(e1_exact=False, family="st", estimator="analytic"):
    return (E1_EXACT if e1_exact else 0) | FAMILIES[family] | ESTIMATORS[estimator]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (FP64, no FMA contraction, OpenMP over independent pairs)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "cfust_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Lattice(C.Structure):
    _fields_ = [("M", C.c_int32), ("s", C.c_int32), ("z", C.POINTER(C.c_uint32)),
                ("shift", C.POINTER(C.c_double))]


_lib = None
_D = C.c_double
_PD = C.POINTER(C.c_double)
_I = C.c_int
_I64 = C.c_int64


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        for name in ["orc_norm_cdf", "orc_norm_quantile", "orc_digamma"]:
            getattr(L, name).restype = _D
            getattr(L, name).argtypes = [_D]
        for name in ["orc_gamma_p", "orc_gamma_q", "orc_chi2_quantile", "orc_t_cdf"]:
            getattr(L, name).restype = _D
            getattr(L, name).argtypes = [_D, _D]
        L.orc_ibeta.restype = _D
        L.orc_ibeta.argtypes = [_D, _D, _D, _D]
        L.orc_t1_logpdf.restype = _D
        L.orc_t1_logpdf.argtypes = [_D, _D, _D, _D]
        L.orc_lattice_w.restype = _D
        L.orc_lattice_w.argtypes = [C.POINTER(_Lattice), _I64, _I]
        L.orc_chi_table.restype = None
        L.orc_chi_table.argtypes = [C.POINTER(_Lattice), _D, _PD]
        L.orc_Tr.restype = _D
        L.orc_Tr.argtypes = [_I, _PD, _PD, _D, C.POINTER(_Lattice), _PD, _PD]
        L.orc_Tr_w.restype = _D
        L.orc_Tr_w.argtypes = [_I, _PD, _PD, _D, C.POINTER(_Lattice), _PD, _PD, _PD, _PD]
        L.orc_logchi_table.restype = None
        L.orc_logchi_table.argtypes = [C.POINTER(_Lattice), _D, _PD]
        L.orc_derive.restype = _I
        L.orc_derive.argtypes = [_I, _I, _PD, _PD, _D, _PD, _PD, _PD, _PD, _PD]
        L.orc_pair.restype = _I
        L.orc_pair.argtypes = [_I, _I, _PD, _PD, _PD, _PD, _PD, _D, _D, C.POINTER(_Lattice),
                               _PD, _PD, _PD, _PD, _PD, _PD, _PD]
        L.orc_estep.restype = _I
        L.orc_estep.argtypes = [_I64, _I, _I, _I, _PD, _PD, _PD, _PD, _PD, _PD, C.POINTER(_Lattice),
                                _I, _I, _PD, _PD, _PD, _PD]
        L.orc_estep_b.restype = _I
        L.orc_estep_b.argtypes = [_I64, _I, _I, _I, _PD, _PD, _PD, _PD, _PD, _PD, C.POINTER(_Lattice),
                                  _I, _I, _PD, _PD, _PD, _PD, _PD]
        L.orc_set_tie_flip.restype = None
        L.orc_set_tie_flip.argtypes = [_I]
        L.orc_mstep.restype = _I
        L.orc_mstep.argtypes = [_I, _I, _I, _D, _PD, _PD, _PD, _PD, _PD, _PD, _D, _D, _I]
        L.orc_pair_sn.restype = _I
        L.orc_pair_sn.argtypes = [_I, _I, _PD, _PD, _PD, _PD, _PD, _D, C.POINTER(_Lattice), _PD, _PD, _PD, _PD]
        L.orc_aitken_stop.restype = _I
        L.orc_aitken_stop.argtypes = [_D, _D, _D, _D]
        L.orc_fit.restype = _I
        L.orc_fit.argtypes = [_I64, _I, _I, _I, _PD, _PD, _PD, _PD, _PD, _PD, C.POINTER(_Lattice),
                              _I, _I, _I, _D, _D, _D, _PD, C.POINTER(_I), C.POINTER(_I)]
        L.orc_k_stats.restype = _I
        L.orc_k_stats.argtypes = [_I, _I]
        _U64 = C.c_uint64
        _PI32 = C.POINTER(C.c_int32)
        L.orc_splitmix64.restype = _U64
        L.orc_splitmix64.argtypes = [_U64]
        L.orc_random_label.restype = _I
        L.orc_random_label.argtypes = [_U64, _I64, _I64, _I]
        L.orc_random_partition.restype = _I
        L.orc_random_partition.argtypes = [_I64, _I, _I, _U64, _I, _I, _PI32]
        L.orc_kmeans.restype = _I
        L.orc_kmeans.argtypes = [_I64, _I, _I, _PD, _U64, _I, _PI32, _PD]
        L.orc_partition_params.restype = _I
        L.orc_partition_params.argtypes = [_I64, _I, _I, _I, _PD, _PI32, _D, _PD, _PD, _PD, _PD, _PD]
        L.orc_init_select.restype = _I
        L.orc_init_select.argtypes = [_I64, _I, _I, _I, _PD, _I, _PI32, C.POINTER(_Lattice), _I, _I, _I, _PD,
                                      C.POINTER(_I), _PD, _PD, _PD, _PD, _PD]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_PD)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class Lattice:
    """Holds the lattice inputs (z, shift) alive for the C side."""

    def __init__(self, M: int, z, shift):
        self.z = np.ascontiguousarray(np.asarray(z, dtype=np.uint32))
        self.shift = _f64(shift)
        self.M = int(M)
        self.s = int(len(self.z)) if M > 0 else 0
        self.c = _Lattice(self.M, self.s, self.z.ctypes.data_as(C.POINTER(C.c_uint32)), _p(self.shift))

    @property
    def ptr(self):
        return C.byref(self.c)


def _nt(nthreads):
    return int(nthreads) if nthreads else (os.cpu_count() or 1)


# --------------------------------------------------------------------- scalar special functions
def norm_cdf(x): return lib().orc_norm_cdf(float(x))
def norm_quantile(u): return lib().orc_norm_quantile(float(u))
def gamma_p(a, x): return lib().orc_gamma_p(float(a), float(x))
def gamma_q(a, x): return lib().orc_gamma_q(float(a), float(x))
def chi2_quantile(w, m): return lib().orc_chi2_quantile(float(w), float(m))
def t_cdf(x, m): return lib().orc_t_cdf(float(x), float(m))
def t1_logpdf(x, loc, s2, m): return lib().orc_t1_logpdf(float(x), float(loc), float(s2), float(m))
def digamma(x): return lib().orc_digamma(float(x))
def ibeta(a, b, x, xc=None): return lib().orc_ibeta(float(a), float(b), float(x), float(1.0 - x if xc is None else xc))
def aitken_stop(l2, l1, l0, tol): return bool(lib().orc_aitken_stop(float(l2), float(l1), float(l0), float(tol)))
def k_stats(p, q): return lib().orc_k_stats(int(p), int(q))


def lattice_w(lat: Lattice, l: int, k: int) -> float:
    return lib().orc_lattice_w(lat.ptr, int(l), int(k))


def chi_table(lat: Lattice, m: float) -> np.ndarray:
    out = np.empty(lat.M)
    lib().orc_chi_table(lat.ptr, float(m), _p(out))
    return out


def logchi_table(lat: Lattice, m: float) -> np.ndarray:
    out = np.empty(lat.M)
    lib().orc_logchi_table(lat.ptr, float(m), _p(out))
    return out


def Tr(b, S, m, lat: Lattice | None = None, chi_s: np.ndarray | None = None, return_gap=False):
    """T_r(b; 0, S, m) by the chi-normal SOV on the lattice (r = len(b))."""
    b = _f64(b).ravel()
    r = len(b)
    S = _f64(S).reshape(r, r)
    gap = np.array([np.inf])
    if r >= 2:
        assert lat is not None
        if chi_s is None:
            chi_s = chi_table(lat, m)
        chi_s = _f64(chi_s)
        v = lib().orc_Tr(r, _p(b), _p(S), float(m), lat.ptr, _p(chi_s), _p(gap))
    else:
        v = lib().orc_Tr(r, _p(b), _p(S), float(m), None, None, _p(gap))
    return (v, gap[0]) if return_gap else v


def derive(sigma, delta, nu):
    sigma = _f64(sigma)
    p = sigma.shape[0]
    delta = _f64(delta).reshape(p, -1)
    q = delta.shape[1]
    L = np.zeros((p, p)); A = np.zeros((max(q, 1), p)); Lam = np.zeros((max(q, 1), max(q, 1)))
    ld = np.zeros(1); ka = np.zeros(1)
    rc = lib().orc_derive(p, q, _p(sigma), _p(delta), float(nu), _p(L), _p(A), _p(Lam), _p(ld), _p(ka))
    return rc, {"L": L, "A": A[:q], "Lambda": Lam[:q, :q], "logdet": ld[0], "kappa": ka[0]}


def pair(y, mu, sigma, delta, nu, lat: Lattice | None, e1_exact: bool = False, family: str = "st"):
    """One (observation, component) pair: dict(logf_noprior, e1me2, e2, e3, e4).
    e1_exact: e1 = E[log W | y] on T0's lattice points (reading R2') instead of reading A5.
    family "sn": the skew-normal limit (CFUSN, nu = inf; reading F1); nu is ignored."""
    y = _f64(y); mu = _f64(mu); p = len(y)
    delta = _f64(delta).reshape(p, -1); q = delta.shape[1]
    rc, dv = derive(sigma, delta, nu)
    assert rc == OK, rc
    m0 = nu + p
    use_lat = lat is not None and (q >= 2 or (e1_exact and q >= 1))
    tabs = [chi_table(lat, m0 + k) if use_lat else np.zeros(1) for k in range(3)]
    lv = logchi_table(lat, m0) if (e1_exact and q >= 1) else None
    out = np.zeros(3 + q + q * q)
    gap = np.array([np.inf])
    A = _f64(dv["A"]) if q else np.zeros(1)
    Lam = _f64(dv["Lambda"]) if q else np.zeros(1)
    if family == "sn":
        ones = np.ones(lat.M if (lat is not None and q >= 2) else 1)
        rc = lib().orc_pair_sn(p, q, _p(y), _p(mu), _p(dv["L"]), _p(A), _p(Lam), float(dv["logdet"]),
                               lat.ptr if lat is not None else None, _p(ones), _p(out), _p(gap), None)
        assert rc == OK, rc
        return {"logf": out[0], "e1me2": out[1], "e2": out[2], "e3": out[3:3 + q],
                "e4": out[3 + q:].reshape(q, q), "gap": gap[0]}
    rc = lib().orc_pair(p, q, _p(y), _p(mu), _p(dv["L"]), _p(A), _p(Lam), float(nu), float(dv["kappa"]),
                        lat.ptr if lat is not None else None, _p(tabs[0]), _p(tabs[1]), _p(tabs[2]),
                        _p(lv) if lv is not None else None, _p(out), _p(gap), None)
    assert rc == OK, rc
    return {"logf": out[0], "e1me2": out[1], "e2": out[2], "e3": out[3:3 + q],
            "e4": out[3 + q:].reshape(q, q), "gap": gap[0]}


def _params(params: dict, g: int, p: int, q: int):
    return (_f64(params["pi"]).reshape(g), _f64(params["mu"]).reshape(g, p),
            _f64(params["sigma"]).reshape(g, p, p),
            _f64(params["delta"]).reshape(g, p, q) if q > 0 else np.zeros(1),
            _f64(params["nu"]).reshape(g))


def set_tie_flip(on: bool):
    """Reading A14 harness: sort near-tied reordering keys (within 1e-12) in the opposite order."""
    lib().orc_set_tie_flip(1 if on else 0)


def estep(y, params: dict, q: int, lat: Lattice | None, nthreads=None, pairs=False, gaps=False,
          e1_exact: bool = False, family: str = "st", estimator: str = "analytic", bounds=False,
          tie_flip=False):
    """Full E-step.  Returns dict(stats [g*K+1], loglik, pairs [n,g,4+q+q*q] optional,
    gaps [n,g] (smallest reordering-key gap), bounds [n,g,q+q*q] (running error bounds of e3/e4,
    analytic estimator)).  tie_flip: evaluate near-tied orders reversed (reading A14)."""
    y = _f64(y)
    n, p = y.shape
    g = len(params["pi"])
    pi, mu, sg, de, nu = _params(params, g, p, q)
    K = k_stats(p, q)
    stats = np.zeros(g * K + 1)
    ll = np.zeros(1)
    po = np.zeros((n, g, 4 + q + q * q)) if pairs else None
    gp = np.full((n, g), np.inf) if gaps else None
    bd = np.zeros((n, g, max(q + q * q, 1))) if bounds else None
    if tie_flip:
        set_tie_flip(True)
    try:
        rc = lib().orc_estep_b(n, p, q, g, _p(y), _p(pi), _p(mu), _p(sg), _p(de), _p(nu),
                               lat.ptr if lat is not None else None, _nt(nthreads),
                               _flags(e1_exact, family, estimator),
                               _p(po) if pairs else None, _p(stats), _p(ll), _p(gp) if gaps else None,
                               _p(bd) if bounds else None)
    finally:
        if tie_flip:
            set_tie_flip(False)
    out = {"rc": rc, "stats": stats, "loglik": ll[0]}
    if bounds:
        out["bounds"] = bd[..., :q + q * q]
    if pairs:
        out["pairs"] = po
    if gaps:
        out["gaps"] = gp
    return out


def mstep(stats, params: dict, p: int, q: int, n_total: float, nu_lo=0.1, nu_hi=1000.0, family: str = "st"):
    g = len(params["pi"])
    pi, mu, sg, de, nu = [a.copy() for a in _params(params, g, p, q)]
    st = _f64(stats)
    rc = lib().orc_mstep(p, q, g, float(n_total), _p(st), _p(pi), _p(mu), _p(sg), _p(de), _p(nu),
                         float(nu_lo), float(nu_hi), FAMILIES[family])
    out = {"pi": pi, "mu": mu, "sigma": sg, "delta": de.reshape(g, p, q) if q > 0 else np.zeros((g, p, 0)),
           "nu": nu}
    return rc, out


def fit(y, params: dict, q: int, lat: Lattice | None, max_iter: int, tol: float = 0.0,
        nthreads=None, nu_lo=0.1, nu_hi=1000.0, e1_exact: bool = False, family: str = "st",
        estimator: str = "analytic"):
    y = _f64(y)
    n, p = y.shape
    g = len(params["pi"])
    pi, mu, sg, de, nu = [a.copy() for a in _params(params, g, p, q)]
    trace = np.zeros(max_iter + 1)
    ni = C.c_int(0); cv = C.c_int(0)
    rc = lib().orc_fit(n, p, q, g, _p(y), _p(pi), _p(mu), _p(sg), _p(de), _p(nu),
                       lat.ptr if lat is not None else None, _nt(nthreads), _flags(e1_exact, family, estimator),
                       int(max_iter),
                       float(tol),
                       float(nu_lo), float(nu_hi), _p(trace), C.byref(ni), C.byref(cv))
    params_out = {"pi": pi, "mu": mu, "sigma": sg,
                  "delta": de.reshape(g, p, q) if q > 0 else np.zeros((g, p, 0)), "nu": nu}
    return {"rc": rc, "params": params_out, "trace": trace[:ni.value + 1], "n_iter": ni.value,
            "converged": bool(cv.value)}


# --------------------------------------------------------------------- Alg. 1 (NEXT-1), readings I1-I4
def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def random_partition(n: int, p: int, g: int, seed: int, l: int, m: int):
    """(attempt, labels[n]) of candidate l (reading I1)."""
    lab = np.zeros(n, dtype=np.int32)
    a = lib().orc_random_partition(int(n), int(p), int(g), C.c_uint64(seed), int(l), int(m), _i32p(lab))
    return a, lab


def kmeans(y, g: int, seed: int, iters: int):
    """(rc, labels[n], centres[g, p]) by reading I2."""
    y = _f64(y)
    n, p = y.shape
    lab = np.zeros(n, dtype=np.int32)
    cen = np.zeros((g, p))
    rc = lib().orc_kmeans(n, p, int(g), _p(y), C.c_uint64(seed), int(iters), _i32p(lab), _p(cen))
    return rc, lab, cen


def partition_params(y, labels, g: int, q: int, n_total=None):
    """(rc, Psi^(0)) from a hard partition (reading I3)."""
    y = _f64(y)
    n, p = y.shape
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
    out = {"pi": np.zeros(g), "mu": np.zeros((g, p)), "sigma": np.zeros((g, p, p)),
           "delta": np.zeros((g, p, max(q, 1))), "nu": np.zeros(g)}
    rc = lib().orc_partition_params(n, p, int(q), int(g), _p(y), _i32p(lab), float(n_total or n), _p(out["pi"]),
                                    _p(out["mu"]), _p(out["sigma"]), _p(out["delta"]), _p(out["nu"]))
    out["delta"] = out["delta"][:, :, :q].copy() if q > 0 else np.zeros((g, p, 0))
    return rc, out


def init_select(y, labels, g: int, q: int, lat: Lattice | None, burn_in: int = 0, nthreads=None,
                family: str = "st"):
    """Alg. 1 lines 3-12 (readings I3, I4): dict(rc, loglik0[m], best, params)."""
    y = _f64(y)
    n, p = y.shape
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
    m = lab.shape[0]
    ll = np.zeros(m)
    best = C.c_int(-1)
    out = {"pi": np.zeros(g), "mu": np.zeros((g, p)), "sigma": np.zeros((g, p, p)),
           "delta": np.zeros((g, p, max(q, 1))), "nu": np.zeros(g)}
    rc = lib().orc_init_select(n, p, int(q), int(g), _p(y), int(m), _i32p(lab), lat.ptr if lat is not None else None,
                               _nt(nthreads), FAMILIES[family], int(burn_in), _p(ll), C.byref(best), _p(out["pi"]),
                               _p(out["mu"]),
                               _p(out["sigma"]), _p(out["delta"]), _p(out["nu"]))
    out["delta"] = out["delta"][:, :, :q].copy() if q > 0 else np.zeros((g, p, 0))
    return {"rc": rc, "loglik0": ll, "best": best.value, "params": out}
