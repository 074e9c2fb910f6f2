"""B200-native FM-CFUST EM hot path (arXiv 2005.06848) — thin Python binding over libcfust.so.

Argument marshalling only: every step of the EM iteration runs in the CUDA kernels behind the
C ABI declared in ``include/cfust.h``.  There is no CPU fallback: if the extension is missing
or no CUDA device is present, calls raise.

    em = CfustEM(y, g=3, q=4, init=params, lattice=(M, z, shift))
    ll = em.iterate()            # one EM iteration (E-step + reduce [+ NCCL] + M-step)
    res = em.fit(max_iter=20)    # Aitken-stopped fit when tol > 0 (Alg. 4)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import (CFUST_EDIM, CFUST_EEMPTY, CFUST_EINVAL, CFUST_EMIXPROP, CFUST_ENCCL,  # noqa: F401
                      CFUST_ENOTPD, CFUST_EUNDERFLOW, CFUST_ECUDA, CfustError, Opts, Params, Result, lib)

__all__ = ["CfustEM", "CfustError", "k_stats", "nccl_unique_id", "eval_special", "lib"]

SPECIAL = {"phi": 0, "phiinv": 1, "exp": 2, "log": 3, "t_cdf": 4, "chi2_quantile": 5, "digamma": 6, "sqrt": 7,
           "trigamma": 8, "lgamma": 9, "phi_xt": 10, "phiinv_xt": 11, "exp_xt": 12}


def eval_special(name: str, x, aux: float = 0.0) -> np.ndarray:
    """Evaluate one of the device special functions (diagnostic; the code the kernels inline)."""
    xs = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    ys = np.empty_like(xs)
    rc = lib().cfust_eval_special(SPECIAL[name], _dptr(xs), _dptr(ys), len(xs), float(aux))
    if rc != 0:
        raise CfustError(rc, f"cfust_eval_special({name})")
    return ys


def k_stats(p: int, q: int) -> int:
    return int(lib().cfust_k_stats(int(p), int(q)))


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = lib().cfust_nccl_unique_id(buf)
    if rc != 0:
        raise CfustError(rc, "ncclGetUniqueId failed")
    return bytes(buf)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class CfustEM:
    """One rank's EM context (its data shard on one GPU)."""

    def __init__(self, y, g: int, q: int, init: dict, lattice=None, *, n_total: int | None = None,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None, device: int = -1,
                 timing: bool = False, nu_lo: float = 0.1, nu_hi: float = 1000.0, e1_exact: bool = False,
                 global_offset: int = 0, family: str = "st", estimator: str = "analytic"):
        L = lib()
        self._keep = []
        on_dev = hasattr(y, "data_ptr") and getattr(y, "is_cuda", False)
        if on_dev:
            assert y.dtype.__str__() == "torch.float64" and y.is_contiguous() and y.dim() == 2
            n, p = int(y.shape[0]), int(y.shape[1])
            yptr = C.cast(C.c_void_p(y.data_ptr()), C.POINTER(C.c_double))
            self._keep.append(y)
        else:
            yh = _f64(y)
            n, p = yh.shape
            yptr = _dptr(yh)
            self._keep.append(yh)
        self.n, self.p, self.g, self.q = int(n), int(p), int(g), int(q)
        self.K = k_stats(p, q)
        prm = self._params_struct(init)
        opts = Opts()
        if lattice is not None and (q >= 2 or ((e1_exact or estimator == "direct") and q >= 1)):
            M, z, sh = lattice
            zz = np.ascontiguousarray(np.asarray(z, dtype=np.uint32))
            ss = _f64(sh)
            self._keep += [zz, ss]
            opts.lattice_m = int(M)
            opts.lattice_z = zz.ctypes.data_as(C.POINTER(C.c_uint32))
            opts.lattice_shift = _dptr(ss)
        opts.nu_lo, opts.nu_hi = float(nu_lo), float(nu_hi)
        opts.y_on_device = 1 if on_dev else 0
        opts.device = int(device)
        opts.rank, opts.world = int(rank), int(world)
        if nccl_id is not None:
            idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            self._keep.append(idbuf)
            opts.nccl_id = C.cast(idbuf, C.c_void_p)
        opts.n_total = int(n_total) if n_total else 0
        opts.timing = 1 if timing else 0
        opts.e1_exact = 1 if e1_exact else 0
        opts.global_offset = int(global_offset)
        opts.family = {"st": 0, "sn": 1}[family]   # skew-t (CFUST) / skew-normal (CFUSN; q = 0: Gaussian)
        opts.estimator = {"analytic": 0, "direct": 1}[estimator]   # truncated moments: O6-O7 / SOV-direct (D1)
        ctx = C.c_void_p()
        rc = L.cfust_em_init(C.byref(ctx), yptr, self.n, self.p, self.g, self.q, C.byref(prm), C.byref(opts))
        if rc != 0:
            raise CfustError(rc, "cfust_em_init failed (see stderr)")
        self._ctx = ctx
        if not on_dev:
            self._keep = self._keep[1:]   # host y was copied

    # ------------------------------------------------------------------ helpers
    def _params_struct(self, d: dict) -> Params:
        g, p, q = self.g, self.p, self.q
        arrs = [_f64(d["pi"]).reshape(g), _f64(d["mu"]).reshape(g, p), _f64(d["sigma"]).reshape(g, p, p),
                _f64(d["delta"]).reshape(g, p, q) if q > 0 else np.zeros(1), _f64(d["nu"]).reshape(g)]
        self._pkeep = arrs
        return Params(*[_dptr(a) for a in arrs])

    def _check(self, rc: int, what: str):
        if rc != 0:
            raise CfustError(rc, f"{what}: {lib().cfust_last_error(self._ctx).decode()}")

    # ------------------------------------------------------------------ API
    def estep(self, want_stats: bool = False):
        ll = C.c_double(0.0)
        st = np.zeros(self.g * self.K + 1) if want_stats else None
        self._check(lib().cfust_estep(self._ctx, C.byref(ll), _dptr(st) if want_stats else None), "cfust_estep")
        return (ll.value, st) if want_stats else ll.value

    def mstep(self):
        self._check(lib().cfust_mstep(self._ctx), "cfust_mstep")

    def iterate(self) -> float:
        ll = C.c_double(0.0)
        self._check(lib().cfust_iterate(self._ctx, C.byref(ll)), "cfust_iterate")
        return ll.value

    def loglik(self) -> float:
        ll = C.c_double(0.0)
        self._check(lib().cfust_loglik(self._ctx, C.byref(ll)), "cfust_loglik")
        return ll.value

    def fit(self, max_iter: int, tol: float = 0.0) -> dict:
        tr = np.zeros(max_iter + 1)
        res = Result()
        res.loglik_trace = _dptr(tr)
        res.trace_cap = max_iter + 1
        self._check(lib().cfust_fit(self._ctx, int(max_iter), float(tol), C.byref(res)), "cfust_fit")
        return {"trace": tr[:res.n_iter + 1].copy(), "n_iter": res.n_iter, "converged": bool(res.converged),
                "wall_time_s": res.wall_time_s, "params": self.params()}

    def params(self) -> dict:
        g, p, q = self.g, self.p, self.q
        out = {"pi": np.zeros(g), "mu": np.zeros((g, p)), "sigma": np.zeros((g, p, p)),
               "delta": np.zeros((g, p, q)), "nu": np.zeros(g)}
        prm = Params(_dptr(out["pi"]), _dptr(out["mu"]), _dptr(out["sigma"]),
                     _dptr(out["delta"]) if q > 0 else None, _dptr(out["nu"]))
        self._check(lib().cfust_get_params(self._ctx, C.byref(prm)), "cfust_get_params")
        return out

    def set_params(self, d: dict):
        prm = self._params_struct(d)
        self._check(lib().cfust_set_params(self._ctx, C.byref(prm)), "cfust_set_params")

    def set_data(self, y):
        if hasattr(y, "data_ptr") and getattr(y, "is_cuda", False):
            self._keep.append(y)
            self._check(lib().cfust_set_data(self._ctx, C.cast(C.c_void_p(y.data_ptr()), C.POINTER(C.c_double)), 1),
                        "cfust_set_data")
        else:
            yh = _f64(y)
            assert yh.shape == (self.n, self.p)
            self._check(lib().cfust_set_data(self._ctx, _dptr(yh), 0), "cfust_set_data")

    def pairs(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        W = 4 + self.q + self.q * self.q
        out = np.zeros((len(idx), self.g, W))
        self._check(lib().cfust_get_pairs(self._ctx, idx.ctypes.data_as(C.POINTER(C.c_int64)), len(idx),
                                          _dptr(out)), "cfust_get_pairs")
        return out

    def predict(self):
        """(labels[n], tau[n, g], loglik) at the current Psi: MAP component and responsibilities."""
        lab = np.zeros(self.n, dtype=np.int32)
        tau = np.zeros((self.n, self.g))
        ll = C.c_double(0.0)
        self._check(lib().cfust_predict(self._ctx, lab.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(tau), C.byref(ll)),
                    "cfust_predict")
        return lab, tau, ll.value

    def init_partitions(self, m: int, seed: int, kmeans_iters: int = 50, want_labels: bool = True):
        """Alg. 1 step 1 (readings I1, I2): candidate 0 k-means, 1..m-1 random; labels [m, n]."""
        out = np.zeros((m, self.n), dtype=np.int32) if want_labels else None
        self._check(lib().cfust_init_partitions(self._ctx, int(m), C.c_uint64(seed), int(kmeans_iters),
                                                out.ctypes.data_as(C.POINTER(C.c_int32)) if want_labels else None),
                    "cfust_init_partitions")
        return out

    def init_select(self, m: int, labels=None, burn_in: int = 0):
        """Alg. 1 steps 2-12 (readings I3, I4): (loglik0[m], best); installs the winner's Psi."""
        ll = np.zeros(m)
        best = C.c_int32(-1)
        lab = None
        if labels is not None:
            lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
            assert lab.shape == (m, self.n)
        self._check(lib().cfust_init_select(self._ctx, int(m), lab.ctypes.data_as(C.POINTER(C.c_int32))
                                            if lab is not None else None, int(burn_in), _dptr(ll), C.byref(best)),
                    "cfust_init_select")
        return ll, int(best.value)

    def timing(self, reset: bool = False):
        ms = np.zeros(4)
        cnt = np.zeros(4, dtype=np.int64)
        self._check(lib().cfust_get_timing(self._ctx, _dptr(ms), cnt.ctypes.data_as(C.POINTER(C.c_int64)),
                                           1 if reset else 0), "cfust_get_timing")
        return ms, cnt

    @property
    def stream_ptr(self) -> int:
        return int(lib().cfust_stream(self._ctx) or 0)

    @property
    def launch_count(self) -> int:
        return int(lib().cfust_launch_count(self._ctx))

    def close(self):
        if getattr(self, "_ctx", None):
            lib().cfust_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
