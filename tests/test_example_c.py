"""examples/cfust_fit.c: the C ABI used from plain C (no Python in the process).  The CPU test
compiles and links it against libcfust.so; the GPU test runs it on a cfg1-shaped problem and checks
its log-likelihood trace equals the Python binding's (same library, same inputs -> same bits)."""
import os
import subprocess

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2005_06848_b200")


def _compile(tmp_path):
    exe = str(tmp_path / "cfust_fit")
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", os.path.join(ROOT, "examples", "cfust_fit.c"),
                    "-I" + os.path.join(ROOT, "include"), "-L" + PKG, "-lcfust", "-Wl,-rpath," + PKG,
                    "-o", exe], check=True)
    return exe


def test_example_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(PKG, "libcfust.so")):
        pytest.skip("libcfust.so not built")
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("config", [1, 2])
def test_example_trace_matches_binding(tmp_path, config):
    import paper_2005_06848_b200 as cf
    exe = _compile(tmp_path)
    prob = str(tmp_path / "problem.bin")
    n = 2000
    subprocess.run(["python", os.path.join(ROOT, "examples", "write_problem.py"), "--config", str(config),
                    "--n", str(n), prob], check=True, cwd=ROOT)
    out = subprocess.run([exe, prob, "5"], check=True, capture_output=True, text=True).stdout
    trace_c = np.array([float(l.split("=")[1]) for l in out.splitlines() if l.startswith("loglik[")])
    cfg = synth.with_n(synth.CONFIGS[config], n)
    y, init, _ = synth.make_problem(cfg)
    em = cf.CfustEM(y, cfg.g, cfg.q, init, synth.lattice_inputs(cfg))
    tr = em.fit(5)["trace"]
    assert len(trace_c) == len(tr)
    # printed with %.10f: equal to the printed precision
    assert np.allclose(trace_c, tr, rtol=0, atol=1e-9)
    sizes = [int(v) for v in out.splitlines()[-1].split(":")[1].split()]
    assert sum(sizes) == n and len(sizes) == cfg.g
