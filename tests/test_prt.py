"""NEXT-4: the Table-1 scaling harness (scripts/prt.py).  Exact check against the paper's own
rows: PRT_m = (T_1 - T_m)/T_1 x 100 recomputed from Table 1's time columns reproduces its
printed time-reduction columns to the printed 2 decimals (reading A22)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import prt  # noqa: E402


def test_paper_table1_prt_recomputed():
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "table1_prt.json")))
    rows = d["rows"]
    r1, m1 = rows[0][1], rows[0][3]
    for m, rt, rp, mt, mp in rows[1:]:
        assert abs(round(prt.prt(r1, rt), 2) - rp) <= 0.0100001, (m, prt.prt(r1, rt), rp)
        assert abs(round(prt.prt(m1, mt), 2) - mp) <= 0.0100001, (m, prt.prt(m1, mt), mp)
    # the paper's observations: 49% / 34% at m = 2; 67% / 64% at m = 4
    r, mm = prt.paper_rows()
    assert round(r[1][2]) == 49 and round(mm[1][2]) == 34 and round(r[3][2]) == 67 and round(mm[3][2]) == 64


def test_harness_on_bench_lines(tmp_path):
    lines = [{"metric": "x", "n_gpus": g, "ms_per_step": t} for g, t in [(1, 100.0), (2, 51.0), (4, 26.0), (8, 13.5)]]
    lines.append({"impl": "reference", "n_gpus": 1, "ms_per_step": 5000.0})   # ignored
    f = tmp_path / "scale.json"
    f.write_text("\n".join(json.dumps(l) for l in lines))
    rows = prt.table(prt.load_bench([str(f)]))
    assert [r[0] for r in rows] == [1, 2, 4, 8]
    assert abs(rows[1][2] - 49.0) < 1e-12 and abs(rows[3][3] - 100 / (8 * 13.5)) < 1e-12
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "prt.py"), str(f)], capture_output=True,
                         text=True)
    assert out.returncode == 0 and "PRT" in out.stdout
