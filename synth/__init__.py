"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no densities, no T_q, no
E-/M-step): it only draws data, initial parameters and the lattice inputs
(generating vector z and the seed-defined shift) that BOTH sides receive as
inputs.  Recipe = BASELINE.json ``configs`` with readings A18/A19.

The paper's own workload is the AIS data set (n=202, p=11, g=2);
it is not available here and these synthetic CFUST mixtures stand in for it.
"""
from __future__ import annotations

import dataclasses
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    p: int
    q: int
    g: int
    M: int            # lattice points (0 when q <= 1: no lattice needed)
    iters: int
    delta_lim: float  # Delta entries ~ U(-delta_lim, delta_lim)
    nu_lo: float
    nu_hi: float
    pi_kind: str      # "uniform" | "dirichlet2" | "dirichlet1"
    mu_kind: str      # "line3" | "normal9" | "grid4"
    data_seed: int
    init_seed: int
    lattice_seed: int


# BASELINE.json configs[0..4]; seeds per SURVEY.md §8(d).
CONFIGS = {
    1: Config("cfg1", 1_000, 2, 2, 2, 1024, 10, 2.0, 4.0, 20.0, "uniform", "line3", 1001, 3001, 2001),
    2: Config("cfg2", 100_000, 4, 4, 3, 2048, 20, 2.0, 4.0, 20.0, "dirichlet2", "line3", 1002, 3002, 2002),
    3: Config("cfg3", 4_000_000, 8, 0, 5, 0, 10, 0.0, 3.0, 30.0, "uniform", "normal9", 1003, 3003, 2003),
    4: Config("cfg4", 1_000_000, 6, 6, 4, 4096, 5, 3.0, 4.0, 12.0, "uniform", "line3", 1004, 3004, 2004),
    5: Config("cfg5", 10_000_000, 3, 3, 8, 2048, 5, 2.0, 4.0, 20.0, "dirichlet1", "grid4", 1005, 3005, 2005),
}


def with_n(cfg: Config, n: int) -> Config:
    """Same generator and shape, different n (reduced-n parity protocol)."""
    return dataclasses.replace(cfg, n=int(n))


def with_(cfg: Config, **kw) -> Config:
    return dataclasses.replace(cfg, **kw)


# ----------------------------------------------------------------------------- parameters
def make_truth(cfg: Config) -> dict:
    """True mixture parameters (reading A18)."""
    rng = np.random.default_rng(cfg.data_seed)
    p, q, g = cfg.p, cfg.q, cfg.g
    if cfg.pi_kind == "uniform":
        pi = np.full(g, 1.0 / g)
    elif cfg.pi_kind == "dirichlet2":
        pi = rng.dirichlet(np.full(g, 2.0))
    elif cfg.pi_kind == "dirichlet1":
        pi = rng.dirichlet(np.full(g, 1.0))
    else:
        raise ValueError(cfg.pi_kind)
    if cfg.mu_kind == "line3":
        v = rng.standard_normal(p)
        v /= np.linalg.norm(v)
        mu = np.stack([3.0 * i * v for i in range(g)])
    elif cfg.mu_kind == "normal9":
        mu = 3.0 * rng.standard_normal((g, p))
    elif cfg.mu_kind == "grid4":
        assert p == 3 and g <= 64
        pts = np.array([(a, b, c) for a in range(4) for b in range(4) for c in range(4)], dtype=np.float64)
        sel = rng.choice(len(pts), size=g, replace=False)
        mu = 4.0 * pts[sel]
    else:
        raise ValueError(cfg.mu_kind)
    sigma = np.empty((g, p, p))
    for i in range(g):
        A = rng.standard_normal((p, p))
        sigma[i] = A @ A.T + 0.5 * np.eye(p)
    delta = rng.uniform(-cfg.delta_lim, cfg.delta_lim, size=(g, p, q)) if q > 0 else np.zeros((g, p, 0))
    nu = rng.uniform(cfg.nu_lo, cfg.nu_hi, size=g)
    return {"pi": pi, "mu": mu, "sigma": sigma, "delta": delta, "nu": nu}


def perturb(cfg: Config, truth: dict) -> dict:
    """Initial parameters = truth perturbed by 10% noise (reading A19)."""
    rng = np.random.default_rng(cfg.init_seed)
    g, p, q = cfg.g, cfg.p, cfg.q
    mu = truth["mu"] + 0.1 * np.sqrt(np.einsum("gii->gi", truth["sigma"])) * rng.standard_normal((g, p))
    D = 1.0 + 0.1 * rng.uniform(-1, 1, size=(g, p))
    sigma = truth["sigma"] * D[:, :, None] * D[:, None, :]
    delta = truth["delta"] * (1.0 + 0.1 * rng.uniform(-1, 1, size=(g, p, q)))
    nu = truth["nu"] * (1.0 + 0.1 * rng.uniform(-1, 1, size=g))
    pi = truth["pi"] * (1.0 + 0.1 * rng.uniform(-1, 1, size=g))
    pi = pi / pi.sum()
    return {"pi": pi, "mu": mu, "sigma": sigma, "delta": delta, "nu": nu}


# ----------------------------------------------------------------------------- data
def sample(cfg: Config, truth: dict, n: int | None = None, return_labels: bool = False):
    """y_j = mu_i + Delta_i |U0| + U1, U0 ~ t_q, U1 ~ t_p(0, Sigma_i) sharing W ~ Gamma(nu/2, rate nu/2).

    Row-major (n, p) float64; labels drawn from pi (BASELINE.json configs, reading A18).
    """
    n = cfg.n if n is None else int(n)
    rng = np.random.default_rng(cfg.data_seed + 7919)
    p, q, g = cfg.p, cfg.q, cfg.g
    lab = rng.choice(g, size=n, p=truth["pi"])
    y = np.empty((n, p))
    for i in range(g):
        idx = np.nonzero(lab == i)[0]
        m = len(idx)
        if m == 0:
            continue
        nu = truth["nu"][i]
        w = rng.gamma(shape=nu / 2.0, scale=2.0 / nu, size=m)
        sw = 1.0 / np.sqrt(w)
        L = np.linalg.cholesky(truth["sigma"][i])
        u1 = (rng.standard_normal((m, p)) @ L.T) * sw[:, None]
        yi = truth["mu"][i][None, :] + u1
        if q > 0:
            u0 = np.abs(rng.standard_normal((m, q))) * sw[:, None]
            yi = yi + u0 @ truth["delta"][i].T
        y[idx] = yi
    y = np.ascontiguousarray(y)
    return (y, lab) if return_labels else y


def make_problem(cfg: Config, n: int | None = None) -> tuple[np.ndarray, dict, dict]:
    truth = make_truth(cfg)
    y = sample(cfg, truth, n)
    init = perturb(cfg, truth)
    return y, init, truth


# ----------------------------------------------------------------------------- lattice inputs
_Z_CACHE: dict | None = None


def lattice_z(M: int, s: int) -> np.ndarray:
    """Generating vector (first s entries) from the committed CBC table (make_lattice_table.py)."""
    global _Z_CACHE
    if _Z_CACHE is None:
        with open(os.path.join(_HERE, "lattice_z.json")) as f:
            _Z_CACHE = json.load(f)
    if str(M) not in _Z_CACHE["z"]:
        raise ValueError(f"no generating vector for M={M}")
    z = _Z_CACHE["z"][str(M)]
    if s > len(z):
        raise ValueError(f"s={s} > table s_max={len(z)}")
    return np.asarray(z[:max(s, 1)], dtype=np.uint32)


def lattice_shift(seed: int, s: int) -> np.ndarray:
    """Seed-defined shift in (0,1): odd multiples of 2^-53, so x = frac(k/M + shift) is never
    exactly 0 or 1/2 (reading A11/A15)."""
    rng = np.random.default_rng(seed)
    k = rng.integers(0, 1 << 52, size=max(s, 1), dtype=np.int64)
    return (2.0 * k.astype(np.float64) + 1.0) / float(1 << 53)


def lattice_dims(q: int) -> int:
    """Chi-normal SOV needs q coordinates for T_q (one chi radius + q-1 normal steps); T_1 is closed form."""
    return q if q >= 2 else 0


def lattice_inputs(cfg: Config, e1_exact: bool = False, direct: bool = False) -> tuple[int, np.ndarray, np.ndarray]:
    """(M, z, shift).  e1_exact with q = 1 needs the one chi coordinate (reading R2'); the SOV-direct
    estimator (reading D1) needs q + 1 coordinates."""
    if direct and cfg.q >= 1:
        M = cfg.M or 1024
        return M, lattice_z(M, cfg.q + 1), lattice_shift(cfg.lattice_seed, cfg.q + 1)
    s = lattice_dims(cfg.q)
    if e1_exact and cfg.q == 1:
        M = cfg.M or 1024
        return M, lattice_z(M, 1), lattice_shift(cfg.lattice_seed, 1)
    if s == 0:
        return 0, np.zeros(1, np.uint32), np.zeros(1)
    return cfg.M, lattice_z(cfg.M, s), lattice_shift(cfg.lattice_seed, s)


def k_stats(p: int, q: int) -> int:
    """Sufficient statistics per component: S0,S1,S2(p),S3(p(p+1)/2),S4(q),S5(q(q+1)/2),S6(p*q),S7."""
    return 3 + p + p * (p + 1) // 2 + q + q * (q + 1) // 2 + p * q


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous blocks whose sizes differ by at most one."""
    base, rem = divmod(n, world)
    j0 = rank * base + min(rank, rem)
    return j0, j0 + base + (1 if rank < rem else 0)


__all__ = ["Config", "CONFIGS", "with_n", "with_", "make_truth", "perturb", "sample", "make_problem",
           "lattice_z", "lattice_shift", "lattice_dims", "lattice_inputs", "k_stats", "shard_range"]
