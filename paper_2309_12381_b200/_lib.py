"""ctypes binding of the C ABI declared in include/mpo.h (argument marshalling only).

Every step of the optimizer path runs in the CUDA library; this module only loads it, declares
the signatures and turns status codes into exceptions.  It fails loudly (ImportError at load,
MpoError at call) when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

# status codes (include/mpo.h: mpo_status)
MPO_OK, MPO_EINVAL, MPO_EALIGN, MPO_EDTYPE, MPO_ECUDA, MPO_ENCCL = range(6)
STATUS_NAMES = {0: "MPO_OK", 1: "MPO_EINVAL", 2: "MPO_EALIGN", 3: "MPO_EDTYPE", 4: "MPO_ECUDA", 5: "MPO_ENCCL"}
# dtype / optimizer enums (mpo_dtype, mpo_optim)
MPO_FP16, MPO_BF16, MPO_FP32 = 0, 1, 2
# storage schemes of the residual: code = base | scheme << 4 (include/mpo.h mpo_dtype)
SCHEMES = {"rne": 0, "rtz": 1, "sr": 2, "x8": 3, "x8z": 4}
MPO_SGD, MPO_ADAM = 0, 1
MPO_MAX_HP_GROUPS = 16

# Every entry point include/mpo.h declares (tests/test_boundary.py checks the header agrees).
SYMBOLS = ("mpo_split", "mpo_reconstruct", "mpo_sgd_step", "mpo_adam_step", "mpo_norm_ws_doubles",
           "mpo_fused_backward_hook_step", "mpo_sharded_step", "mpo_last_error", "mpo_build_exact",
           "mpo_launch_count", "mpo_selfcheck_fastmath", "mpo_nvls_sharded_step", "mpo_nvls_alloc_local",
           "mpo_nvls_free_local", "mpo_p2p_sharded_step", "mpo_grad_sumsq", "mpo_sharded_step_grouped",
           "mpo_comm_check", "mpo_hp_block_bytes", "mpo_hp_block_fill", "mpo_step_graphed",
           "mpo_nvls_emulated_step")


class MpoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Tensor(C.Structure):
    """mpo_tensor"""
    _fields_ = [("value", C.c_void_p), ("resid", C.c_void_p), ("grad", C.c_void_p), ("m", C.c_void_p),
                ("v", C.c_void_p), ("n", C.c_int64), ("hp", C.c_int32), ("sr_stream", C.c_int32)]


class SgdHP(C.Structure):
    """mpo_sgd_hp"""
    _fields_ = [("lr", C.c_double), ("momentum", C.c_double), ("dampening", C.c_double),
                ("weight_decay", C.c_double), ("grad_scale", C.c_double), ("nesterov", C.c_int32),
                ("first_step", C.c_int32), ("seed", C.c_uint64), ("clip_value", C.c_double),
                ("skip_nonfinite", C.c_int32), ("norm_ready", C.c_int32)]


class AdamHP(C.Structure):
    """mpo_adam_hp"""
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("grad_scale", C.c_double), ("max_grad_norm", C.c_double),
                ("adamw", C.c_int32), ("_pad", C.c_int32), ("step", C.c_int64), ("seed", C.c_uint64),
                ("clip_value", C.c_double), ("skip_nonfinite", C.c_int32), ("norm_ready", C.c_int32)]


class Segment(C.Structure):
    """mpo_segment"""
    _fields_ = [("start", C.c_int64), ("hp", C.c_int32), ("sr_stream", C.c_int32)]


_libs: dict = {}


def _declare(L):
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_int
    L.mpo_split.argtypes = [D, P, P, P, I64, C.c_uint64, I32, P]
    L.mpo_reconstruct.argtypes = [D, P, P, P, I64, P]
    L.mpo_sgd_step.argtypes = [D, D, C.POINTER(Tensor), I32, C.POINTER(SgdHP), I32, P, P]
    L.mpo_adam_step.argtypes = [D, D, C.POINTER(Tensor), I32, C.POINTER(AdamHP), I32, P, P]
    L.mpo_fused_backward_hook_step.argtypes = [D, D, D, C.POINTER(Tensor), P, P, P]
    L.mpo_sharded_step.argtypes = [D, C.c_size_t, I32, I32, D, P, P, P, P, P, I64, P, P, P]
    L.mpo_sharded_step_grouped.argtypes = [D, C.c_size_t, I32, I32, D, P, P, P, P, P, I64, C.POINTER(Segment), I32,
                                           P, I32, P, P]
    L.mpo_grad_sumsq.argtypes = [D, C.POINTER(Tensor), I32, C.POINTER(C.c_double), I32, P, I32, P]
    L.mpo_comm_check.argtypes = [C.c_size_t]
    L.mpo_hp_block_bytes.argtypes = [D]
    L.mpo_hp_block_bytes.restype = I64
    L.mpo_hp_block_fill.argtypes = [D, P, I32, C.c_uint64, P]
    L.mpo_step_graphed.argtypes = [D, D, D, C.POINTER(Tensor), I32, P, I32, P, P, P, P, P]
    for f in ("mpo_split", "mpo_reconstruct", "mpo_sgd_step", "mpo_adam_step", "mpo_fused_backward_hook_step",
              "mpo_sharded_step", "mpo_sharded_step_grouped", "mpo_grad_sumsq", "mpo_comm_check", "mpo_hp_block_fill",
              "mpo_step_graphed"):
        getattr(L, f).restype = C.c_int
    L.mpo_last_error.restype = C.c_char_p
    L.mpo_last_error.argtypes = []
    L.mpo_build_exact.restype = I32
    L.mpo_launch_count.restype = I64
    L.mpo_norm_ws_doubles.restype = I64
    L.mpo_selfcheck_fastmath.argtypes = [I64, C.c_uint64, P, P]
    L.mpo_selfcheck_fastmath.restype = C.c_int
    L.mpo_nvls_sharded_step.argtypes = [D, I32, I32, D, P, P, P, P, P, P, I64, P, P]
    L.mpo_nvls_sharded_step.restype = C.c_int
    L.mpo_nvls_alloc_local.argtypes = [I64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
    L.mpo_nvls_alloc_local.restype = C.c_int
    L.mpo_nvls_free_local.argtypes = [P, P, I64]
    L.mpo_nvls_free_local.restype = C.c_int
    L.mpo_p2p_sharded_step.argtypes = [D, I32, I32, D, P, P, P, P, P, I64, P, P]
    L.mpo_p2p_sharded_step.restype = C.c_int
    L.mpo_nvls_emulated_step.argtypes = [D, I32, I32, D, P, P, P, P, P, I64, P, P]
    L.mpo_nvls_emulated_step.restype = C.c_int


def load(exact: bool = True):
    """Load libmpo_exact.so (-fmad=false: bit-exact to the CPU oracle; the default of every entry
    point) or libmpo.so (exact=False: FMA contraction, within DESIGN.md R12's tolerance; measured
    0.5-1 % faster on the step, profiles/r02_ab_bulkst_exact.log)."""
    key = bool(exact)
    if key not in _libs:
        path = _build.lib_path(exact)
        override = os.environ.get("MPO_LIB_OVERRIDE")   # A/B experiments only (scripts/ab_variants.py)
        if override:
            path = override
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with `python -m paper_2309_12381_b200._build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(path)
        _declare(L)
        _libs[key] = L
    return _libs[key]


def check(L, status: int):
    if status != MPO_OK:
        raise MpoError(status, L.mpo_last_error().decode())
