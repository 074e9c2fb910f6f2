"""bench.py's roofline constants recompute from the committed ncu captures they name (VERDICT r01
weak #7: nothing typed in by hand): for every entry of profiles/roofline_constants.json, parse its
`source` with scripts/roofline_constants.py's own parser and rebuild flops per pair and DRAM bytes."""
import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _script():
    spec = importlib.util.spec_from_file_location("roofline_constants", os.path.join(ROOT, "scripts", "roofline_constants.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


with open(os.path.join(ROOT, "profiles", "roofline_constants.json")) as _f:
    CONST = json.load(_f)


@pytest.mark.parametrize("name", sorted(CONST))
def test_constants_recompute_from_capture(name):
    e = CONST[name]
    src = os.path.join(ROOT, e["source"])
    assert os.path.exists(src), f"capture {e['source']} is not committed"
    kernel, m = _script().parse(src)
    assert kernel == e["kernel"] and "estep_cfust_kernel" in kernel
    flops = (2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
             + m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
             + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"])
    assert flops / e["pairs"] == pytest.approx(e["flops_per_pair"], rel=1e-12)
    rd, wr = m["dram__bytes_read.sum"] * e["bytes_scale"], m["dram__bytes_write.sum"] * e["bytes_scale"]
    assert rd == pytest.approx(e["dram_read_bytes"], rel=1e-12)
    assert wr == pytest.approx(e["dram_write_bytes"], rel=1e-12, abs=1e-9)
    assert rd + wr == pytest.approx(e["dram_bytes_per_launch"], rel=1e-12)
    # the executed-flop rate under ncu is below the nominal FP64 peak (148 SM x 64 DFMA/clk x 2 x 1.965 GHz)
    assert 0.0 < e["ncu_flop_rate_tflops"] < 37.22496
