"""ctypes declarations for libcfust.so (include/cfust.h).  Loads the in-tree library built by
``python -m paper_2005_06848_b200.build``; fails loudly if it is missing — there is no fallback."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CFUST_LIB") or os.path.join(_HERE, "libcfust.so")   # CFUST_LIB: experiment builds

CFUST_OK, CFUST_EINVAL, CFUST_EDIM, CFUST_EMIXPROP, CFUST_ENOTPD = 0, -1, -2, -3, -4
CFUST_EUNDERFLOW, CFUST_EEMPTY, CFUST_ECUDA, CFUST_ENCCL = -5, -6, -7, -8
_NAMES = {0: "OK", -1: "EINVAL", -2: "EDIM", -3: "EMIXPROP", -4: "ENOTPD", -5: "EUNDERFLOW", -6: "EEMPTY",
          -7: "ECUDA", -8: "ENCCL"}


class CfustError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"CFUST_{_NAMES.get(code, code)} ({code}): {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("pi", C.POINTER(C.c_double)), ("mu", C.POINTER(C.c_double)), ("sigma", C.POINTER(C.c_double)),
                ("delta", C.POINTER(C.c_double)), ("nu", C.POINTER(C.c_double))]


class Opts(C.Structure):
    _fields_ = [("lattice_m", C.c_int32), ("lattice_z", C.POINTER(C.c_uint32)),
                ("lattice_shift", C.POINTER(C.c_double)), ("nu_lo", C.c_double), ("nu_hi", C.c_double),
                ("y_on_device", C.c_int32), ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_id", C.c_void_p), ("n_total", C.c_int64), ("timing", C.c_int32),
                ("e1_exact", C.c_int32), ("global_offset", C.c_int64), ("family", C.c_int32),
                ("estimator", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("n_iter", C.c_int32), ("converged", C.c_int32), ("loglik_trace", C.POINTER(C.c_double)),
                ("trace_cap", C.c_int32), ("wall_time_s", C.c_double)]


# every symbol declared in include/cfust.h (checked by tests/test_abi_symbols.py)
EXPORTS = ["cfust_em_init", "cfust_set_data", "cfust_estep", "cfust_mstep", "cfust_iterate", "cfust_loglik",
           "cfust_fit", "cfust_get_params", "cfust_set_params", "cfust_get_pairs", "cfust_get_timing",
           "cfust_stream", "cfust_launch_count", "cfust_nccl_unique_id", "cfust_eval_special", "cfust_k_stats",
           "cfust_init_partitions", "cfust_init_select", "cfust_predict",
           "cfust_last_error", "cfust_destroy"]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built: run `python -m paper_2005_06848_b200.build` "
                               "(nvcc, sm_100a). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
        L.cfust_em_init.argtypes = [C.POINTER(vp), dp, i64, i32, i32, i32, C.POINTER(Params), C.POINTER(Opts)]
        L.cfust_set_data.argtypes = [vp, dp, i32]
        L.cfust_estep.argtypes = [vp, dp, dp]
        L.cfust_mstep.argtypes = [vp]
        L.cfust_iterate.argtypes = [vp, dp]
        L.cfust_loglik.argtypes = [vp, dp]
        L.cfust_fit.argtypes = [vp, i32, C.c_double, C.POINTER(Result)]
        L.cfust_get_params.argtypes = [vp, C.POINTER(Params)]
        L.cfust_set_params.argtypes = [vp, C.POINTER(Params)]
        L.cfust_get_pairs.argtypes = [vp, C.POINTER(C.c_int64), i64, dp]
        L.cfust_get_timing.argtypes = [vp, dp, C.POINTER(C.c_int64), i32]
        L.cfust_stream.argtypes = [vp]
        L.cfust_stream.restype = vp
        L.cfust_launch_count.argtypes = [vp]
        L.cfust_launch_count.restype = i64
        L.cfust_nccl_unique_id.argtypes = [vp]
        L.cfust_k_stats.argtypes = [i32, i32]
        L.cfust_eval_special.argtypes = [i32, dp, dp, i64, C.c_double]
        pi32 = C.POINTER(C.c_int32)
        L.cfust_init_partitions.argtypes = [vp, i32, C.c_uint64, i32, pi32]
        L.cfust_init_select.argtypes = [vp, i32, pi32, i32, dp, pi32]
        L.cfust_predict.argtypes = [vp, pi32, dp, dp]
        L.cfust_last_error.argtypes = [vp]
        L.cfust_last_error.restype = C.c_char_p
        L.cfust_destroy.argtypes = [vp]
        L.cfust_destroy.restype = None
        for name in ["cfust_em_init", "cfust_set_data", "cfust_estep", "cfust_mstep", "cfust_iterate",
                     "cfust_loglik", "cfust_fit", "cfust_get_params", "cfust_set_params", "cfust_get_pairs",
                     "cfust_get_timing", "cfust_nccl_unique_id", "cfust_k_stats", "cfust_eval_special"]:
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib
