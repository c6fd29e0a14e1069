"""Thin Python binding of include/mpo.h: the same entry points, torch tensors in, pointers out.

Only argument marshalling happens here (pointer/size/enum extraction, hyper-parameter structs,
the current CUDA stream); every step of the path runs in libmpo's kernels.  PyTorch supplies
device memory, streams and process groups.  Citations as in include/mpo.h.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import MPO_ADAM, MPO_BF16, MPO_FP16, MPO_FP32, MPO_SGD, AdamHP, MpoError, Segment, SgdHP, Tensor

_DT = {torch.float16: MPO_FP16, torch.bfloat16: MPO_BF16, torch.float32: MPO_FP32}
_VALUE_VIEW = {torch.float16, torch.bfloat16}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DT[dt]
    except KeyError:
        raise MpoError(_lib.MPO_EDTYPE, f"unsupported dtype {dt}") from None


def format_code(value_dtype: torch.dtype, scheme: str = "rne") -> int:
    """Storage format code (include/mpo.h mpo_dtype) of a 16-bit value dtype under a scheme:
    'rne' (default), 'rtz' (round-to-zero + uint16 extra bits), 'sr' (fp16 stochastic rounding),
    'x8' (8 extra bits, int8 residual), 'x8z' (the paper's fp16+8: round-to-zero value + the next
    8 bits truncated, uint8 residual)."""
    if value_dtype not in _VALUE_VIEW:
        raise MpoError(_lib.MPO_EDTYPE, f"value dtype must be fp16/bf16, got {value_dtype}")
    if scheme not in _lib.SCHEMES:
        raise MpoError(_lib.MPO_EDTYPE, f"unknown scheme {scheme!r}")
    if scheme == "sr" and value_dtype != torch.float16:
        raise MpoError(_lib.MPO_EDTYPE, "stochastic rounding is defined for fp16 (13 extra bits + the un-round bit)")
    return dtype_code(value_dtype) | (_lib.SCHEMES[scheme] << 4)


def resid_dtype(scheme: str = "rne") -> torch.dtype:
    """Container dtype of the residual: int16 (rne, sr; rtz holds uint16 bit patterns), int8 (x8),
    uint8 (x8z)."""
    return {"x8": torch.int8, "x8z": torch.uint8}.get(scheme, torch.int16)


def step_seed(seed: int, step: int) -> int:
    """Per-step key of the stochastic-rounding draws (any fixed mixing works; this is the one the
    optimizers use)."""
    return (int(seed) * 0x9E3779B97F4A7C15 + int(step)) & 0xFFFFFFFFFFFFFFFF


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_cur_dev = getattr(torch._C, "_cuda_getDevice", None)


def _stream(stream) -> int:
    if stream is None:
        # the current stream's handle straight from torch's C API (~10x cheaper per call than
        # building a torch.cuda.Stream object; the same handle)
        if _raw_stream is not None and _cur_dev is not None:
            return _raw_stream(_cur_dev())
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise MpoError(_lib.MPO_EINVAL, "tensor is not on a CUDA device (no CPU path)")
    if not t.is_contiguous():
        raise MpoError(_lib.MPO_EINVAL, "tensor is not contiguous")
    return t.data_ptr()


def _lib_of(exact: bool):
    return _lib.load(exact)


# ------------------------------------------------------------------------------------------
# Hyper-parameter structs
# ------------------------------------------------------------------------------------------
@dataclass
class SgdParams:
    lr: float
    momentum: float = 0.0
    dampening: float = 0.0
    weight_decay: float = 0.0
    grad_scale: float = 1.0
    nesterov: bool = False
    first_step: bool = False
    seed: int = 0
    clip_value: float = 0.0
    skip_nonfinite: bool = False
    norm_ready: bool = False

    def c(self) -> SgdHP:
        return SgdHP(self.lr, self.momentum, self.dampening, self.weight_decay, self.grad_scale,
                     int(self.nesterov), int(self.first_step), int(self.seed), float(self.clip_value),
                     int(self.skip_nonfinite), int(self.norm_ready))


@dataclass
class AdamParams:
    lr: float
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    grad_scale: float = 1.0
    max_grad_norm: float = 0.0
    adamw: bool = True
    step: int = 1
    seed: int = 0
    clip_value: float = 0.0
    skip_nonfinite: bool = False
    norm_ready: bool = False

    def c(self) -> AdamHP:
        return AdamHP(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay, self.grad_scale,
                      self.max_grad_norm, int(self.adamw), 0, int(self.step), int(self.seed),
                      float(self.clip_value), int(self.skip_nonfinite), int(self.norm_ready))


def _hp_array(hps, kind):
    if isinstance(hps, (SgdParams, AdamParams)):
        hps = [hps]
    arr = (kind * len(hps))()
    for i, h in enumerate(hps):
        arr[i] = h.c()
    return arr, len(hps)


# ------------------------------------------------------------------------------------------
# Multi-tensor table
# ------------------------------------------------------------------------------------------
class TensorTable:
    """A packed mpo_tensor array ("one only stream of values").

    Rows are (value, resid, grad, m, v, hp_index); the tensors are referenced, not copied, and the
    row pointers are cached so a step does not rebuild the table.  ``set_grads`` refreshes only
    the gradient pointers."""

    def __init__(self, values: Sequence[torch.Tensor], resids: Sequence[torch.Tensor],
                 grads: Sequence[Optional[torch.Tensor]], ms: Sequence[Optional[torch.Tensor]],
                 vs: Sequence[Optional[torch.Tensor]], hp_index: Optional[Sequence[int]] = None,
                 scheme: str = "rne", sr_streams: Optional[Sequence[int]] = None):
        n = len(values)
        if not (len(resids) == len(grads) == len(ms) == len(vs) == n):
            raise MpoError(_lib.MPO_EINVAL, "table columns differ in length")
        self.values, self.resids, self.ms, self.vs = list(values), list(resids), list(ms), list(vs)
        self.hp_index = list(hp_index) if hp_index is not None else [0] * n
        self.arr = (Tensor * max(n, 1))()
        self.nt = n
        self.scheme = scheme
        self.vdt = format_code(values[0].dtype, scheme) if n else MPO_FP16
        rdt = resid_dtype(scheme)
        for i in range(n):
            v, r = values[i], resids[i]
            if v.dtype not in _VALUE_VIEW or r.dtype != rdt or v.numel() != r.numel():
                raise MpoError(_lib.MPO_EDTYPE, f"tensor {i}: value must be fp16/bf16 and resid {rdt} of equal size")
            if format_code(v.dtype, scheme) != self.vdt:
                raise MpoError(_lib.MPO_EDTYPE, f"tensor {i}: mixed value dtypes in one table")
            row = self.arr[i]
            row.value = _ptr(v)
            row.resid = _ptr(r)
            row.m = _ptr(ms[i])
            row.v = _ptr(vs[i])
            row.n = v.numel()
            row.hp = self.hp_index[i]
            row.sr_stream = int(sr_streams[i]) if sr_streams is not None else i
        self.gdt = None
        self.set_grads(grads)

    def set_grads(self, grads: Sequence[Optional[torch.Tensor]]):
        gdt = None
        for i, g in enumerate(grads):
            if g is None:
                raise MpoError(_lib.MPO_EINVAL, f"tensor {i}: missing gradient")
            if g.numel() != self.arr[i].n:
                raise MpoError(_lib.MPO_EINVAL, f"tensor {i}: gradient size mismatch")
            c = dtype_code(g.dtype)
            if gdt is None:
                gdt = c
            elif c != gdt:
                raise MpoError(_lib.MPO_EDTYPE, f"tensor {i}: mixed gradient dtypes in one table")
            self.arr[i].grad = _ptr(g)
        # pointers only: the table must not keep gradients alive (hook / set_to_none training frees them)
        self.grad_ptrs = [g.data_ptr() for g in grads]
        self.gdt = gdt if gdt is not None else self.vdt


# ------------------------------------------------------------------------------------------
# Entry points (same names as the C ABI)
# ------------------------------------------------------------------------------------------
def mpo_split(w: torch.Tensor, fmt: torch.dtype, value: Optional[torch.Tensor] = None,
              resid: Optional[torch.Tensor] = None, stream=None, exact: bool = True, scheme: str = "rne",
              seed: int = 0, sr_stream: int = 0):
    """fp32 -> (16-bit value, residual) under a storage scheme."""
    if w.dtype != torch.float32:
        raise MpoError(_lib.MPO_EDTYPE, "split input must be fp32")
    if value is None:
        value = torch.empty(w.shape, dtype=fmt, device=w.device)
    if resid is None:
        resid = torch.empty(w.shape, dtype=resid_dtype(scheme), device=w.device)
    if resid.dtype != resid_dtype(scheme):
        raise MpoError(_lib.MPO_EDTYPE, f"resid must be {resid_dtype(scheme)} for scheme {scheme!r}")
    L = _lib_of(exact)
    _lib.check(L, L.mpo_split(format_code(value.dtype, scheme), _ptr(w), _ptr(value), _ptr(resid), w.numel(),
                              int(seed), int(sr_stream), _stream(stream)))
    return value, resid


def mpo_reconstruct(value: torch.Tensor, resid: torch.Tensor, out: Optional[torch.Tensor] = None,
                    stream=None, exact: bool = True, scheme: str = "rne") -> torch.Tensor:
    """(16-bit value, residual) -> fp32."""
    if out is None:
        out = torch.empty(value.shape, dtype=torch.float32, device=value.device)
    if value.numel() != resid.numel() or value.numel() != out.numel():
        raise MpoError(_lib.MPO_EINVAL, "size mismatch")
    if resid.dtype != resid_dtype(scheme):
        raise MpoError(_lib.MPO_EDTYPE, f"resid must be {resid_dtype(scheme)} for scheme {scheme!r}")
    L = _lib_of(exact)
    _lib.check(L, L.mpo_reconstruct(format_code(value.dtype, scheme), _ptr(value), _ptr(resid), _ptr(out),
                                    value.numel(), _stream(stream)))
    return out


def _check_ws(norm_ws, exact):
    if norm_ws is not None and (norm_ws.dtype != torch.float64 or norm_ws.numel() < norm_ws_doubles(exact)):
        raise MpoError(_lib.MPO_EINVAL, "norm_ws must be a float64 tensor of norm_ws_doubles() entries")


def mpo_sgd_step(table: TensorTable, hps, norm_ws: Optional[torch.Tensor] = None, stream=None, exact: bool = True):
    """Residual-compensated SGD(-momentum) step over a table; skip_nonfinite needs norm_ws."""
    # one group: a pointer to the struct itself (no array built)
    arr, nhp = (C.byref(hps.c()), 1) if isinstance(hps, SgdParams) else _hp_array(hps, SgdHP)
    L = _lib_of(exact)
    _check_ws(norm_ws, exact)
    _lib.check(L, L.mpo_sgd_step(table.vdt, table.gdt, table.arr, table.nt, arr, nhp, _ptr(norm_ws), _stream(stream)))


def mpo_adam_step(table: TensorTable, hps, norm_ws: Optional[torch.Tensor] = None, stream=None,
                  exact: bool = True):
    """Residual-compensated Adam/AdamW step over a table; clipping needs norm_ws."""
    arr, nhp = (C.byref(hps.c()), 1) if isinstance(hps, AdamParams) else _hp_array(hps, AdamHP)
    L = _lib_of(exact)
    _check_ws(norm_ws, exact)
    _lib.check(L, L.mpo_adam_step(table.vdt, table.gdt, table.arr, table.nt, arr, nhp, _ptr(norm_ws),
                                  _stream(stream)))


def mpo_fused_backward_hook_step(kind: int, vdt: int, gdt: int, one: Tensor, hp, stream=None,
                                 exact: bool = True, norm_ws: Optional[torch.Tensor] = None):
    """One parameter's step from its post-accumulate-grad hook.  ``one`` is an
    mpo_tensor row, ``hp`` an SgdHP / AdamHP struct (kept by the caller); norm_ws is needed for
    skip_nonfinite (its last entry accumulates the sums of squares over the backward)."""
    L = _lib_of(exact)
    _lib.check(L, L.mpo_fused_backward_hook_step(kind, vdt, gdt, C.byref(one), C.byref(hp), _ptr(norm_ws),
                                                 _stream(stream)))


def mpo_sharded_step(kind: int, comm_ptr: int, rank: int, world: int, value_flat: torch.Tensor,
                     grad_flat: torch.Tensor, resid_shard: torch.Tensor, m_shard: Optional[torch.Tensor],
                     v_shard: Optional[torch.Tensor], hp, norm_ws: Optional[torch.Tensor] = None, stream=None,
                     exact: bool = True, scheme: str = "rne", segments=None):
    """Data-parallel sharded step: RS(grad) -> shard update -> AG(value) (BASELINE north_star (c)).

    ``hp``: one hyper-parameter set, or a list of groups together with ``segments``, a list of
    (start in the shard, group index, sr_stream) pieces partitioning this rank's shard
    (mpo_sharded_step_grouped)."""
    if grad_flat.dtype != value_flat.dtype or grad_flat.numel() != value_flat.numel():
        raise MpoError(_lib.MPO_EINVAL, "grad_flat must match value_flat in dtype and size")
    L = _lib_of(exact)
    vdt = format_code(value_flat.dtype, scheme)
    if segments is None and not isinstance(hp, (list, tuple)):
        chp = hp.c() if hasattr(hp, "c") else hp
        _lib.check(L, L.mpo_sharded_step(kind, comm_ptr, rank, world, vdt, _ptr(value_flat), _ptr(grad_flat),
                                         _ptr(resid_shard), _ptr(m_shard), _ptr(v_shard), value_flat.numel(),
                                         C.byref(chp), _ptr(norm_ws), _stream(stream)))
        return
    hps = list(hp) if isinstance(hp, (list, tuple)) else [hp]
    segments = segments if segments is not None else [(0, 0, rank)]
    arr, nhp = _hp_array(hps, AdamHP if kind == MPO_ADAM else SgdHP)
    seg = (Segment * len(segments))(*[Segment(int(a), int(h), int(s)) for a, h, s in segments])
    _lib.check(L, L.mpo_sharded_step_grouped(kind, comm_ptr, rank, world, vdt, _ptr(value_flat), _ptr(grad_flat),
                                             _ptr(resid_shard), _ptr(m_shard), _ptr(v_shard), value_flat.numel(),
                                             seg, len(segments), C.cast(arr, C.c_void_p), nhp, _ptr(norm_ws),
                                             _stream(stream)))


def mpo_grad_sumsq(table: TensorTable, grad_scales, norm_ws: torch.Tensor, accumulate: bool = False, stream=None,
                   exact: bool = True):
    """S = sum (f32(g) * grad_scale[group])^2 over a table into norm_ws[0] (``accumulate``: added to it);
    the shared pre-pass of a step spanning several tables (include/mpo.h norm_ready)."""
    gs = (C.c_double * len(grad_scales))(*[float(x) for x in grad_scales])
    L = _lib_of(exact)
    _check_ws(norm_ws, exact)
    _lib.check(L, L.mpo_grad_sumsq(table.gdt, table.arr, table.nt, gs, len(grad_scales), _ptr(norm_ws),
                                   int(bool(accumulate)), _stream(stream)))


def hp_block_bytes(kind: int, exact: bool = True) -> int:
    """Bytes of the per-step hyper-parameter block of mpo_step_graphed."""
    return int(_lib_of(exact).mpo_hp_block_bytes(kind))


def hp_block_fill(kind: int, hps, host_block: torch.Tensor, seq: int = 0, exact: bool = True):
    """Derive this step's kernel scalars from ``hps`` into ``host_block`` (pinned uint8 tensor of
    hp_block_bytes(kind) bytes), tagged with ``seq``; a host function, no CUDA call (include/mpo.h)."""
    arr, nhp = _hp_array(hps, AdamHP if kind == MPO_ADAM else SgdHP)
    if host_block.device.type != "cpu" or host_block.numel() * host_block.element_size() < hp_block_bytes(kind, exact):
        raise MpoError(_lib.MPO_EINVAL, "host_block must be a host tensor of hp_block_bytes() bytes")
    L = _lib_of(exact)
    _lib.check(L, L.mpo_hp_block_fill(kind, C.cast(arr, C.c_void_p), nhp, int(seq), host_block.data_ptr()))


def mpo_step_graphed(kind: int, table: TensorTable, hps, host_block: torch.Tensor, dev_block: torch.Tensor,
                     ack: Optional[torch.Tensor] = None, norm_ws: Optional[torch.Tensor] = None, stream=None,
                     exact: bool = True):
    """A step whose per-step hyper-parameters are copied host_block -> dev_block in stream order and
    read by the kernels from there: capturable once in a CUDA graph, replayed every step after
    hp_block_fill (include/mpo.h mpo_step_graphed).  host_block (and ack: one pinned int64 the
    device echoes the block's sequence number to) must be pinned."""
    if not host_block.is_pinned() or (ack is not None and not ack.is_pinned()):
        raise MpoError(_lib.MPO_EINVAL, "host_block / ack must be pinned (page-locked) host memory")
    arr, nhp = _hp_array(hps, AdamHP if kind == MPO_ADAM else SgdHP)
    L = _lib_of(exact)
    _check_ws(norm_ws, exact)
    _lib.check(L, L.mpo_step_graphed(kind, table.vdt, table.gdt, table.arr, table.nt, C.cast(arr, C.c_void_p), nhp,
                                     host_block.data_ptr(), _ptr(dev_block), None if ack is None else ack.data_ptr(),
                                     _ptr(norm_ws), _stream(stream)))


def mpo_comm_check(comm_ptr: int, exact: bool = True):
    """Raises MpoError(MPO_ENCCL) if the NCCL communicator failed asynchronously (never blocks)."""
    L = _lib_of(exact)
    _lib.check(L, L.mpo_comm_check(comm_ptr))


def mpo_selfcheck_fastmath(pairs: int = 1 << 30, seed: int = 0xB0B, exact: bool = True, stream=None):
    """Fast sqrt/div sequences vs IEEE sqrtf and `/` on the device (diagnostic; see include/mpo.h).
    Returns (sqrt mismatches, div mismatches, sqrt fast-path count, div fast-path count)."""
    counts = torch.zeros(4, dtype=torch.int64, device="cuda")
    L = _lib_of(exact)
    _lib.check(L, L.mpo_selfcheck_fastmath(pairs, seed, _ptr(counts), _stream(stream)))
    return tuple(int(x) for x in counts.cpu())


def mpo_p2p_sharded_step(kind: int, rank: int, world: int, value_peers: Sequence[int], grad_peers: Sequence[int],
                         resid_shard: torch.Tensor, m_shard: Optional[torch.Tensor], v_shard: Optional[torch.Tensor],
                         n_total: int, hp, value_dtype: torch.dtype, stream=None, exact: bool = True,
                         scheme: str = "rne"):
    """The sharded step fused with its collectives over NVLink peer memory (include/mpo.h): one
    kernel reads every rank's gradient shard (P2P), updates, and writes the new values into every
    rank's replica.  value_peers / grad_peers: raw device addresses (ints) of every rank's value
    replica and gradient buffer, mapped into this process (rank order)."""
    if len(value_peers) != world or len(grad_peers) != world:
        raise MpoError(_lib.MPO_EINVAL, "need one value and one gradient address per rank")
    L = _lib_of(exact)
    chp = hp.c() if hasattr(hp, "c") else hp
    vp = (C.c_void_p * world)(*[C.c_void_p(int(a)) for a in value_peers])
    gp = (C.c_void_p * world)(*[C.c_void_p(int(a)) for a in grad_peers])
    _lib.check(L, L.mpo_p2p_sharded_step(kind, rank, world, format_code(value_dtype, scheme), vp, gp,
                                         _ptr(resid_shard), _ptr(m_shard), _ptr(v_shard), n_total, C.byref(chp),
                                         _stream(stream)))


def mpo_nvls_sharded_step(kind: int, rank: int, world: int, vdt: int, value_mc: int, value_uc: int, grad_mc: int,
                          resid_shard: torch.Tensor, m_shard: Optional[torch.Tensor], v_shard: Optional[torch.Tensor],
                          n_total: int, hp, stream=None, exact: bool = True):
    """The sharded step fused with its collectives over NVLink SHARP (include/mpo.h): multicast
    addresses are raw device addresses (ints) of a multicast object every rank bound."""
    L = _lib_of(exact)
    chp = hp.c() if hasattr(hp, "c") else hp
    _lib.check(L, L.mpo_nvls_sharded_step(kind, rank, world, vdt, value_mc, value_uc, grad_mc, _ptr(resid_shard),
                                          _ptr(m_shard), _ptr(v_shard), n_total, C.byref(chp), _stream(stream)))


def mpo_nvls_emulated_step(kind: int, rank: int, world: int, value_peers: Sequence[int], grad_peers: Sequence[int],
                           resid_shard: torch.Tensor, m_shard: Optional[torch.Tensor], v_shard: Optional[torch.Tensor],
                           n_total: int, hp, value_dtype: torch.dtype, stream=None, exact: bool = True,
                           scheme: str = "rne"):
    """The NVLS kernel with its multicast operations emulated over peer addresses (validation on a
    box without a multicast object; include/mpo.h).  Arguments as mpo_p2p_sharded_step."""
    if len(value_peers) != world or len(grad_peers) != world:
        raise MpoError(_lib.MPO_EINVAL, "need one value and one gradient address per rank")
    L = _lib_of(exact)
    chp = hp.c() if hasattr(hp, "c") else hp
    vp = (C.c_void_p * world)(*[C.c_void_p(int(a)) for a in value_peers])
    gp = (C.c_void_p * world)(*[C.c_void_p(int(a)) for a in grad_peers])
    _lib.check(L, L.mpo_nvls_emulated_step(kind, rank, world, format_code(value_dtype, scheme), vp, gp, _ptr(resid_shard),
                                           _ptr(m_shard), _ptr(v_shard), n_total, C.byref(chp), _stream(stream)))


class NvlsLocalBuffer:
    """A single-device multicast object bound to fresh memory (world-1 NVLS runs and tests):
    ``uc`` / ``mc`` are the unicast / multicast device addresses of the same bytes."""

    def __init__(self, nbytes: int, exact: bool = True):
        self._L = _lib_of(exact)
        uc, mc, sz = C.c_void_p(), C.c_void_p(), C.c_int64()
        _lib.check(self._L, self._L.mpo_nvls_alloc_local(nbytes, C.byref(uc), C.byref(mc), C.byref(sz)))
        self.uc, self.mc, self.size = uc.value, mc.value, sz.value

    def free(self):
        if self.uc:
            _lib.check(self._L, self._L.mpo_nvls_free_local(self.uc, self.mc, self.size))
            self.uc = self.mc = None


def norm_ws_doubles(exact: bool = True) -> int:
    return int(_lib_of(exact).mpo_norm_ws_doubles())


def launch_count(exact: bool = True) -> int:
    return int(_lib_of(exact).mpo_launch_count())


def build_exact(exact: bool) -> int:
    return int(_lib_of(exact).mpo_build_exact())
