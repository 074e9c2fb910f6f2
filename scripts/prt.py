"""Table-1-style scaling harness.

The paper reports, per worker count m, the mean total time T_m and the "time reduction"
PRT_m = (T_1 - T_m) / T_1 x 100 (reading A22: the text's "(total time in MATLAB - total time in R)
/ (total time in R)" at PAPER.md:478-480 is garbled; the printed Table 1 values are (T_1 - T_m)/T_1
per implementation, checked exactly by tests/test_prt.py).  Here the workers are B200s: T_G is the
EM-iteration time (bench.py ms_per_step, max over ranks) of the same workload at G GPUs.

    python scripts/prt.py SCALE_r01.json [more bench JSON files or lines ...]
    python scripts/prt.py --paper            # the paper's own rows, recomputed

Prints one row per G: G, ms_per_step, PRT (%), parallel efficiency T_1 / (G T_G).
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def prt(t1: float, tm: float) -> float:
    """Percentage reduction in time against the single-worker baseline (Table 1)."""
    return (t1 - tm) / t1 * 100.0


def table(times: dict[int, float]) -> list[tuple[int, float, float | None, float]]:
    """rows (G, T_G, PRT_G, efficiency) for G in ascending order; T_1 must be present."""
    t1 = times[1]
    return [(g, t, None if g == 1 else prt(t1, t), t1 / (g * t)) for g, t in sorted(times.items())]


def paper_rows():
    with open(os.path.join(ROOT, "tests", "golden", "table1_prt.json")) as f:
        d = json.load(f)
    r = {row[0]: row[1] for row in d["rows"]}
    mt = {row[0]: row[3] for row in d["rows"]}
    return table(r), table(mt)


def load_bench(paths: list[str]) -> dict[int, float]:
    """ms_per_step per n_gpus from bench.py JSON lines (files with one or more lines, or lists)."""
    times: dict[int, float] = {}
    for pth in paths:
        txt = open(pth).read().strip()
        objs = []
        try:
            obj = json.loads(txt)
            objs = obj if isinstance(obj, list) else [obj]
        except json.JSONDecodeError:
            objs = [json.loads(l) for l in txt.splitlines() if l.strip().startswith("{")]
        stack = list(objs)
        while stack:   # bench lines anywhere in the structure (a list, or nested under other keys)
            o = stack.pop()
            if isinstance(o, dict):
                if "n_gpus" in o and "ms_per_step" in o and o.get("impl") != "reference":
                    times[int(o["n_gpus"])] = float(o["ms_per_step"])
                else:
                    stack.extend(o.values())
            elif isinstance(o, list):
                stack.extend(o)
    return times


def main():
    if "--paper" in sys.argv:
        r, m = paper_rows()
        print("m  R_time_s  R_PRT%  | MATLAB_time_s  MATLAB_PRT%")
        for (g, t, p, _), (_, t2, p2, _) in zip(r, m):
            print(f"{g:2d} {t:9.2f} {'--' if p is None else f'{p:6.2f}':>7} | {t2:9.2f} {'--' if p2 is None else f'{p2:6.2f}':>7}")
        return
    times = load_bench(sys.argv[1:])
    if 1 not in times:
        raise SystemExit("need the G = 1 line (T_1) among the inputs")
    print("G  ms_per_step  PRT%   efficiency")
    for g, t, p, e in table(times):
        print(f"{g:2d} {t:11.3f} {'--' if p is None else f'{p:6.2f}':>7} {e:8.3f}")


if __name__ == "__main__":
    main()
