"""ctypes wrapper of the plain-C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs are the only permitted importers.  The product package
paper_2309_12381_b200 never imports this module (tests/test_boundary.py checks it).

Arrays are numpy; 16-bit values travel as uint16 bit patterns, residuals as int16.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# The same source built with -fopenmp: element loops split across threads, nothing else changes
# (bit-identical, tests/test_oracle_omp.py).  Only bench.py's all-core CPU baseline uses it.
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")

FMT = {"fp16": 0, "bf16": 1, "fp32": 2}

CFLAGS = ["-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fno-unsafe-math-optimizations",
          "-fPIC", "-shared", "-Wall"]


def _build_one(out: str, extra) -> str:
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)
    return out


def build(force: bool = False) -> str:
    """Compile liboracle.so (and the OpenMP build liboracle_omp.so) with gcc (building the checker
    is not using it)."""
    if force:
        for f in (_LIB, _LIB_OMP):
            if os.path.exists(f):
                os.unlink(f)
    _build_one(_LIB_OMP, ["-fopenmp"])
    return _build_one(_LIB, [])


class SgdHP(C.Structure):
    _fields_ = [("lr", C.c_double), ("momentum", C.c_double), ("dampening", C.c_double),
                ("weight_decay", C.c_double), ("grad_scale", C.c_double),
                ("nesterov", C.c_int32), ("first_step", C.c_int32), ("clip_value", C.c_double)]


class AdamHP(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double), ("grad_scale", C.c_double),
                ("adamw", C.c_int32), ("step", C.c_int64), ("clip_value", C.c_double)]


_lib = None
_lib_omp = None
_parallel = False


def parallel(on: bool = True, threads: int = 0) -> int:
    """Route the wrappers below through the OpenMP build (``on``) with ``threads`` threads (0: all
    of OpenMP's default, i.e. every core of the affinity mask), or back to the plain build.
    Returns the thread count in effect."""
    global _parallel
    _parallel = bool(on)
    return int(lib().or_threads(int(threads)))


def lib():
    global _lib, _lib_omp
    if _lib is None:
        build()
        _lib = _declare(C.CDLL(_LIB))
        _lib_omp = _declare(C.CDLL(_LIB_OMP))
    return _lib_omp if _parallel else _lib


def _declare(L):
    L.or_fpenv_clear.restype = C.c_uint
    L.or_fpenv_ok.restype = C.c_int
    L.or_rne16.restype = C.c_uint16
    L.or_rne16.argtypes = [C.c_int, C.c_uint32]
    L.or_widen16.restype = C.c_uint32
    L.or_widen16.argtypes = [C.c_int, C.c_uint16]
    P = C.c_void_p
    L.or_split.argtypes = [C.c_int, P, P, P, C.c_int64]
    L.or_reconstruct.argtypes = [C.c_int, P, P, P, C.c_int64]
    L.or_cast16.argtypes = [C.c_int, P, P, C.c_int64]
    L.or_widen.argtypes = [C.c_int, P, P, C.c_int64]
    L.or_sgd_step.argtypes = [C.c_int, C.c_int, P, P, P, P, C.c_int64, C.POINTER(SgdHP)]
    L.or_adam_step.argtypes = [C.c_int, C.c_int, P, P, P, P, P, C.c_int64,
                               C.POINTER(AdamHP), C.c_float]
    L.or_sgd_step_master.argtypes = [C.c_int, P, P, P, C.c_int64, C.POINTER(SgdHP)]
    L.or_adam_step_master.argtypes = [C.c_int, P, P, P, P, C.c_int64, C.POINTER(AdamHP),
                                      C.c_float]
    L.or_sumsq.restype = C.c_double
    L.or_sumsq.argtypes = [C.c_int, P, C.c_int64, C.c_double]
    L.or_clip_coef.restype = C.c_float
    L.or_clip_coef.argtypes = [C.c_double, C.c_double]
    L.or_rtz16.restype = C.c_uint16
    L.or_rtz16.argtypes = [C.c_int, C.c_uint32]
    L.or_sr16.restype = C.c_uint16
    L.or_sr16.argtypes = [C.c_uint32, C.c_uint32]
    L.or_mix64.restype = C.c_uint64
    L.or_mix64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    L.or_split_s.argtypes = [C.c_int, C.c_int, P, P, P, C.c_int64, C.c_uint64, C.c_uint64]
    L.or_reconstruct_s.argtypes = [C.c_int, C.c_int, P, P, P, C.c_int64]
    L.or_sgd_step_s.argtypes = [C.c_int, C.c_int, C.c_int, P, P, P, P, C.c_int64, C.POINTER(SgdHP),
                                C.c_uint64, C.c_uint64]
    L.or_adam_step_s.argtypes = [C.c_int, C.c_int, C.c_int, P, P, P, P, P, C.c_int64, C.POINTER(AdamHP),
                                 C.c_float, C.c_uint64, C.c_uint64]
    L.or_reduce_sum16.argtypes = [C.c_int, C.c_int, P, P, C.c_int64]
    L.or_bytes_per_param.restype = C.c_int
    L.or_bytes_per_param.argtypes = [C.c_int, C.c_int]
    L.or_threads.restype = C.c_int
    L.or_threads.argtypes = [C.c_int]
    L.or_fpenv_clear()
    return L


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _chk(a, dtype):
    assert isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous, (a.dtype, dtype)
    return a


def fpenv_ok() -> bool:
    return bool(lib().or_fpenv_ok())


def rne16(fmt: str, u: int) -> int:
    return lib().or_rne16(FMT[fmt], u)


def widen16(fmt: str, h: int) -> int:
    return lib().or_widen16(FMT[fmt], h)


def split(fmt: str, w: np.ndarray):
    """fp32 -> (value uint16 bits, residual int16)."""
    w = _chk(np.ascontiguousarray(w, dtype=np.float32), np.float32)
    h = np.empty(w.shape, np.uint16)
    r = np.empty(w.shape, np.int16)
    lib().or_split(FMT[fmt], _ptr(w), _ptr(h), _ptr(r), w.size)
    return h, r


def reconstruct(fmt: str, h: np.ndarray, r: np.ndarray) -> np.ndarray:
    h = _chk(np.ascontiguousarray(h, dtype=np.uint16), np.uint16)
    r = _chk(np.ascontiguousarray(r, dtype=np.int16), np.int16)
    assert h.shape == r.shape
    w = np.empty(h.shape, np.float32)
    lib().or_reconstruct(FMT[fmt], _ptr(h), _ptr(r), _ptr(w), h.size)
    return w


def cast16(fmt: str, w: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.float32)
    out = np.empty(w.shape, np.uint16)
    lib().or_cast16(FMT[fmt], _ptr(w), _ptr(out), w.size)
    return out


def widen(fmt: str, h: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16)
    out = np.empty(h.shape, np.float32)
    lib().or_widen(FMT[fmt], _ptr(h), _ptr(out), h.size)
    return out


def _grad_fmt(grad: np.ndarray, gfmt: str):
    if gfmt == "fp32":
        return _chk(grad, np.float32)
    return _chk(grad, np.uint16)


def sgd_step(vfmt, gfmt, value, resid, grad, buf, *, lr, momentum=0.0, dampening=0.0,
             weight_decay=0.0, grad_scale=1.0, nesterov=False, first_step=False, clip_value=0.0):
    """In-place residual-compensated SGD step on one tensor (buf may be None if momentum=0)."""
    _chk(value, np.uint16); _chk(resid, np.int16); _grad_fmt(grad, gfmt)
    if buf is not None:
        _chk(buf, np.float32)
    hp = SgdHP(lr, momentum, dampening, weight_decay, grad_scale, int(nesterov), int(first_step), clip_value)
    lib().or_sgd_step(FMT[vfmt], FMT[gfmt], _ptr(value), _ptr(resid), _ptr(grad), _ptr(buf),
                      value.size, C.byref(hp))


def adam_step(vfmt, gfmt, value, resid, grad, m, v, *, lr, beta1=0.9, beta2=0.999, eps=1e-8,
              weight_decay=0.0, adamw=True, grad_scale=1.0, step=1, clip_coef=None, clip_value=0.0):
    """In-place residual-compensated Adam/AdamW step on one tensor."""
    _chk(value, np.uint16); _chk(resid, np.int16); _grad_fmt(grad, gfmt)
    _chk(m, np.float32); _chk(v, np.float32)
    hp = AdamHP(lr, beta1, beta2, eps, weight_decay, grad_scale, int(adamw), int(step), clip_value)
    cc = -1.0 if clip_coef is None else float(clip_coef)
    lib().or_adam_step(FMT[vfmt], FMT[gfmt], _ptr(value), _ptr(resid), _ptr(grad), _ptr(m),
                       _ptr(v), value.size, C.byref(hp), cc)


def sgd_step_master(gfmt, w, grad, buf, *, lr, momentum=0.0, dampening=0.0, weight_decay=0.0,
                    grad_scale=1.0, nesterov=False, first_step=False, clip_value=0.0):
    _chk(w, np.float32); _grad_fmt(grad, gfmt)
    hp = SgdHP(lr, momentum, dampening, weight_decay, grad_scale, int(nesterov), int(first_step), clip_value)
    lib().or_sgd_step_master(FMT[gfmt], _ptr(w), _ptr(grad), _ptr(buf), w.size, C.byref(hp))


def adam_step_master(gfmt, w, grad, m, v, *, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                     weight_decay=0.0, adamw=True, grad_scale=1.0, step=1, clip_coef=None, clip_value=0.0):
    _chk(w, np.float32); _grad_fmt(grad, gfmt)
    hp = AdamHP(lr, beta1, beta2, eps, weight_decay, grad_scale, int(adamw), int(step), clip_value)
    cc = -1.0 if clip_coef is None else float(clip_coef)
    lib().or_adam_step_master(FMT[gfmt], _ptr(w), _ptr(grad), _ptr(m), _ptr(v), w.size,
                              C.byref(hp), cc)


def sumsq(gfmt, grad, grad_scale=1.0) -> float:
    _grad_fmt(grad, gfmt)
    return lib().or_sumsq(FMT[gfmt], _ptr(grad), grad.size, grad_scale)


def reduce_sum16(fmt: str, grads) -> np.ndarray:
    """R15: the P2P sharded step's reduction over ranks: each rank's 16-bit gradient
    widened exactly to binary32 and summed in binary32 in rank order."""
    gs = [_chk(np.ascontiguousarray(g, dtype=np.uint16), np.uint16) for g in grads]
    n = gs[0].size
    assert all(g.size == n for g in gs)
    arr = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    out = np.empty(n, np.float32)
    lib().or_reduce_sum16(FMT[fmt], len(gs), arr, _ptr(out), n)
    return out


def clip_coef(sumsq_: float, max_norm: float) -> float:
    return lib().or_clip_coef(sumsq_, max_norm)


def bytes_per_param(scheme: str, optim: str) -> int:
    s = {"amp": 0, "ours_fused_backward": 1, "ours_multi_tensor": 2}[scheme]
    o = {"sgd_momentum": 0, "adam": 1}[optim]
    return lib().or_bytes_per_param(s, o)


# ---- paper variants of the storage scheme (oracle.c "Paper variants") ----
SCHEME = {"rne": 0, "rtz": 1, "sr": 2, "x8": 3, "x8z": 4}
RESID_DTYPE = {"rne": np.int16, "rtz": np.uint16, "sr": np.int16, "x8": np.int8, "x8z": np.uint8}


def rtz16(fmt: str, u: int) -> int:
    return lib().or_rtz16(FMT[fmt], u)


def sr16(u: int, rnd: int) -> int:
    return lib().or_sr16(u, rnd)


def mix64(seed: int, stream: int, index: int) -> int:
    return lib().or_mix64(seed, stream, index)


def split_s(scheme: str, fmt: str, w: np.ndarray, seed: int = 0, stream: int = 0):
    """fp32 -> (value uint16 bits, residual in the scheme's dtype)."""
    w = _chk(np.ascontiguousarray(w, dtype=np.float32), np.float32)
    h = np.empty(w.shape, np.uint16)
    r = np.empty(w.shape, RESID_DTYPE[scheme])
    lib().or_split_s(SCHEME[scheme], FMT[fmt], _ptr(w), _ptr(h), _ptr(r), w.size, seed, stream)
    return h, r


def reconstruct_s(scheme: str, fmt: str, h: np.ndarray, r: np.ndarray) -> np.ndarray:
    h = _chk(np.ascontiguousarray(h, dtype=np.uint16), np.uint16)
    r = _chk(np.ascontiguousarray(r), RESID_DTYPE[scheme])
    w = np.empty(h.shape, np.float32)
    lib().or_reconstruct_s(SCHEME[scheme], FMT[fmt], _ptr(h), _ptr(r), _ptr(w), h.size)
    return w


def sgd_step_s(scheme, vfmt, gfmt, value, resid, grad, buf, *, lr, momentum=0.0, dampening=0.0,
               weight_decay=0.0, grad_scale=1.0, nesterov=False, first_step=False, seed=0, stream=0,
               clip_value=0.0):
    _chk(value, np.uint16); _chk(resid, RESID_DTYPE[scheme]); _grad_fmt(grad, gfmt)
    hp = SgdHP(lr, momentum, dampening, weight_decay, grad_scale, int(nesterov), int(first_step), clip_value)
    lib().or_sgd_step_s(SCHEME[scheme], FMT[vfmt], FMT[gfmt], _ptr(value), _ptr(resid), _ptr(grad), _ptr(buf),
                        value.size, C.byref(hp), seed, stream)


def adam_step_s(scheme, vfmt, gfmt, value, resid, grad, m, v, *, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                weight_decay=0.0, adamw=True, grad_scale=1.0, step=1, clip_coef=None, seed=0, stream=0,
                clip_value=0.0):
    _chk(value, np.uint16); _chk(resid, RESID_DTYPE[scheme]); _grad_fmt(grad, gfmt)
    _chk(m, np.float32); _chk(v, np.float32)
    hp = AdamHP(lr, beta1, beta2, eps, weight_decay, grad_scale, int(adamw), int(step), clip_value)
    cc = -1.0 if clip_coef is None else float(clip_coef)
    lib().or_adam_step_s(SCHEME[scheme], FMT[vfmt], FMT[gfmt], _ptr(value), _ptr(resid), _ptr(grad), _ptr(m),
                         _ptr(v), value.size, C.byref(hp), cc, seed, stream)
