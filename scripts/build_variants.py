"""Build experiment variants of libcfust (occupancy / polynomial scheme) side by side."""
import subprocess
import sys
import os
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_06848_b200 import build as B  # noqa: E402

VARIANTS = {v.split("=", 1)[0]: v.split("=", 1)[1].split(",") for v in sys.argv[1:]}


def one(name, flags):
    out = os.path.join(B.HERE, f"libcfust_{name}.so")
    r = subprocess.run(B.nvcc_cmd(out, [f"-D{f}" for f in flags if f]), capture_output=True, text=True)
    regs = [l for l in r.stderr.split("\n") if "registers" in l]
    return name, r.returncode, r.stderr[-300:] if r.returncode else ""


with ThreadPoolExecutor(4) as ex:
    for name, rc, err in ex.map(lambda kv: one(*kv), VARIANTS.items()):
        print(name, rc, err)
