"""Build libcfust.so in-tree for sm_100a (nvcc; no JIT, no torch extension machinery)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcfust.so")
SOURCES = ["cfust_kernels.cu", "cfust_init.cu", "cfust_abi.cu"]
HEADERS = ["cfust_device.cuh", "cfust_internal.h", "cfust_special.cuh", "cfust_coeffs.h"]


def nccl_paths() -> tuple[str, str]:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        cands += [os.path.join(p, "nccl") for p in spec.submodule_search_locations]
    cands.append(os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                              "site-packages", "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h not found (expected the torch-bundled nvidia/nccl package)")


def nvcc_cmd(out: str = LIB, extra: list[str] | None = None) -> list[str]:
    inc, lib = nccl_paths()
    return (["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
             f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}", f"-I{inc}"]
            + (extra or [])
            + [os.path.join(CSRC, s) for s in SOURCES]
            + ["-o", out, f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}"])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "cfust.h")]
    return any(os.path.getmtime(d) > t for d in deps)


PEAK_LIB = os.path.join(HERE, "libfp64peak.so")


def build_peak(force: bool = False) -> str:
    src = os.path.join(CSRC, "fp64_peak.cu")
    if force or not os.path.exists(PEAK_LIB) or os.path.getmtime(PEAK_LIB) < os.path.getmtime(src):
        tmp = PEAK_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                               "-shared", src, "-o", tmp])
        os.replace(tmp, PEAK_LIB)
    return PEAK_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    build_peak(force)
    if force or stale():
        tmp = LIB + f".tmp{os.getpid()}"
        r = subprocess.run(nvcc_cmd(tmp), capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        with open(os.path.join(HERE, "ptxas.log"), "w") as f:
            f.write(r.stderr)
        if verbose:
            print(r.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
