"""CPU-side checks of the boundary: libcfust.so loads and exports every symbol include/cfust.h
declares (no compute calls without a GPU); the Python binding declares the same names."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2005_06848_b200 import build as B
    return B.build()


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "cfust.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cfust_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_north_star_calls():
    names = _header_functions()
    for n in ["cfust_em_init", "cfust_estep", "cfust_mstep", "cfust_loglik", "cfust_fit"]:
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in _header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (cfust_[a-z_0-9]+)\b", out))
    assert set(_header_functions()) <= exported


def test_binding_matches_header(libpath):
    from paper_2005_06848_b200 import _native
    assert sorted(_native.EXPORTS) == _header_functions()


def test_k_stats_cpu(libpath):
    from paper_2005_06848_b200 import _native
    import synth
    L = _native.lib()
    for p, q in [(2, 2), (4, 4), (8, 0), (6, 6), (3, 3)]:
        assert L.cfust_k_stats(p, q) == synth.k_stats(p, q)
    # BASELINE/SURVEY vector sizes g*K+1 for cfgs 1..5
    assert [g * synth.k_stats(p, q) + 1 for p, q, g in [(2, 2, 2), (4, 4, 3), (8, 0, 5), (6, 6, 4), (3, 3, 8)]] == \
        [35, 142, 236, 373, 241]


def test_no_device_fails_loudly(libpath):
    """Without a GPU the product path must fail (CFUST_ECUDA), never fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2005_06848_b200 as cf
    import synth
    cfg = synth.with_n(synth.CONFIGS[1], 10)
    y, init, _ = synth.make_problem(cfg)
    with pytest.raises(cf.CfustError) as e:
        cf.CfustEM(y, cfg.g, cfg.q, init, synth.lattice_inputs(cfg))
    assert e.value.code == cf.CFUST_ECUDA
    assert np.isfinite(y).all()


def test_product_never_imports_oracle():
    """The product package and its sources share no code with oracle/."""
    pkg = os.path.join(ROOT, "paper_2005_06848_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "cfust_oracle" not in txt, f
