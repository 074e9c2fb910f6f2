"""Build the committed rank-1 lattice generating-vector table (reading A12).

The paper never states how T_q is evaluated (PAPER.md:424-425 only says "the
same set of commands"); BASELINE.json fixes "a seed-defined randomized rank-1
lattice of M points".  The generating vector z is an INPUT shared by the oracle
and the CUDA path (neither computes it), produced once by this script with a
plain component-by-component (CBC) search and committed as
``synth/lattice_z.json``.

CBC criterion (standard shift-averaged worst-case error in the weighted Korobov
space with smoothness alpha=2, product weights gamma_j = 1/j^2):

    e^2(z_1..z_s) = -1 + (1/M) sum_{k=0}^{M-1} prod_{j<=s} (1 + gamma_j * omega({k z_j / M}))
    omega(x) = 2 pi^2 (x^2 - x + 1/6)

z_1 = 1; for j >= 2 pick the odd z in [1, M/2) minimising e^2 given z_1..z_{j-1}
(ties -> smallest z).  The construction is dimension-extensible, so the first r
entries serve every T_r with r <= S_MAX.

Run:  python synth/make_lattice_table.py   (about a minute for M up to 2^16)
"""
from __future__ import annotations

import json
import os

import numpy as np

M_LIST = [1 << k for k in range(10, 17)]   # 2^10 .. 2^16 (SURVEY.md §8(b) limits)
S_MAX = 7                                  # q <= 6: chi-normal SOV needs <= q coordinates; the SOV-direct estimator q+1


def omega_table(M: int) -> np.ndarray:
    x = np.arange(M, dtype=np.float64) / M
    return 2.0 * np.pi ** 2 * (x * x - x + 1.0 / 6.0)


def cbc(M: int, s: int) -> list[int]:
    om = omega_table(M)
    k = np.arange(M, dtype=np.int64)
    prod = np.ones(M, dtype=np.float64)
    z = [1]
    prod *= 1.0 + 1.0 * om[(k * 1) % M]
    cands = np.arange(1, M // 2, 2, dtype=np.int64)
    for j in range(2, s + 1):
        gamma = 1.0 / (j * j)
        best = None
        chunk = max(1, (1 << 24) // M)
        for c0 in range(0, len(cands), chunk):
            cz = cands[c0:c0 + chunk]
            idx = (cz[:, None] * k[None, :]) % M
            cost = (prod[None, :] * (1.0 + gamma * om[idx])).sum(axis=1)
            i = int(np.argmin(cost))
            if best is None or cost[i] < best[0]:
                best = (float(cost[i]), int(cz[i]))
        zj = best[1]
        z.append(zj)
        prod *= 1.0 + gamma * om[(k * zj) % M]
    return z


def main() -> None:
    table = {"criterion": "CBC, Korobov alpha=2, gamma_j=1/j^2, odd z < M/2, z_1=1",
             "s_max": S_MAX, "z": {}}
    for M in M_LIST:
        table["z"][str(M)] = cbc(M, S_MAX)
        print(M, table["z"][str(M)], flush=True)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lattice_z.json")
    with open(out, "w") as f:
        json.dump(table, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
