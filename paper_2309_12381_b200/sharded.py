"""Data-parallel sharded residual optimizer (BASELINE.json north_star (c); not in the paper, which
lists distributed training as future work).

Layout: all parameters live in one flat 16-bit buffer, each parameter at
an offset aligned to 8 elements (16 B), the total padded to a multiple of 8*world.  Every rank
holds the whole value buffer (replicated) and a whole flat gradient buffer (the params' .grad
are views of it), but only its 1/world shard of residual, m and v.  One step is
``mpo_sharded_step``: NCCL reduce-scatter of the 16-bit grads over NVLink -> residual-compensated
update of the local shard -> NCCL all-gather of the 16-bit values only.

``ShardLayout`` is pure host logic (tested with gloo on CPU); ``ShardedResidualOptimizer`` drives
the CUDA library through torch's NCCL communicator.
"""
from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import api
from ._lib import MPO_ADAM, MPO_SGD, MpoError

ALIGN = 8   # elements: 16 B for 16-bit data, so every parameter view is 16-byte aligned


@dataclass
class ShardLayout:
    sizes: List[int]
    world: int
    align: int = ALIGN      # 16 for the int8-residual (X8) formats: every piece 16-B aligned

    def __post_init__(self):
        if self.world < 1:
            raise ValueError("world must be >= 1")
        a = self.align
        offs, o = [], 0
        for n in self.sizes:
            offs.append(o)
            o += (n + a - 1) // a * a
        q = a * self.world
        self.offsets = offs
        self.used = o
        self.total = (o + q - 1) // q * q
        self.shard = self.total // self.world

    def shard_range(self, rank: int):
        return rank * self.shard, (rank + 1) * self.shard

    def views(self, flat: torch.Tensor, shapes: Sequence[torch.Size]):
        return [flat[o:o + n].view(s) for o, n, s in zip(self.offsets, self.sizes, shapes)]

    def segments(self, rank: int, hp_index: Sequence[int]):
        """mpo_segment table of ``rank``'s shard for per-parameter hyper-parameter groups: runs of
        consecutive parameter pieces with the same group become one segment (padding goes with the
        preceding piece), starting at 0; segment k draws stochastic-rounding numbers from stream
        rank + world*k (one segment: stream = rank, as mpo_sharded_step)."""
        segs = []
        for i, _, start, _ in self.owner_slices(rank):
            h = int(hp_index[i])
            if not segs:
                segs.append([0, h])
            elif segs[-1][1] != h:
                segs.append([start, h])
        if not segs:
            segs = [[0, 0]]
        return [(a, h, rank + self.world * k) for k, (a, h) in enumerate(segs)]

    def owner_slices(self, rank: int):
        """(param index, start within param, start within shard, length) of the parameter pieces
        that fall in ``rank``'s shard (padding excluded)."""
        lo, hi = self.shard_range(rank)
        out = []
        for i, (o, n) in enumerate(zip(self.offsets, self.sizes)):
            a, b = max(o, lo), min(o + n, hi)
            if a < b:
                out.append((i, a - o, a - lo, b - a))
        return out


def nccl_comm_ptr(group=None) -> int:
    """Borrow torch's NCCL communicator for ``group`` (created eagerly by a warm-up collective)."""
    import torch.distributed as dist
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    t = torch.zeros(1, device="cuda")
    dist.all_reduce(t, group=pg)   # makes sure the communicator exists before borrowing it
    torch.cuda.synchronize()
    return int(pg._get_backend(torch.device("cuda"))._comm_ptr())


def _symm_empty(n: int, dtype: torch.dtype, device) -> torch.Tensor:
    import torch.distributed._symmetric_memory as symm
    return symm.empty(n, dtype=dtype, device=device)


def _rendezvous(t: torch.Tensor, group):
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    pg = group if group is not None else dist.group.WORLD
    name = pg.group_name
    try:
        return symm.rendezvous(t, name)
    except Exception:
        if not hasattr(symm, "enable_symm_mem_for_group"):
            raise
        symm.enable_symm_mem_for_group(name)   # older torch needs the opt-in
        return symm.rendezvous(t, name)


def _peer_addrs(h, t: torch.Tensor, rank: int) -> List[int]:
    """Device addresses of every rank's copy of the symmetric tensor t, in rank order."""
    ptrs = list(h.buffer_ptrs)
    off = t.data_ptr() - int(ptrs[rank])
    return [int(p) + off for p in ptrs]


def _shard_state_dict(opt, layout_desc):
    """Checkpoint of one rank's sharded optimizer state (R17): this rank's residual / m / v shard in
    their own dtypes, the step count, the hyper-parameters and what identifies the layout.  The
    16-bit values are the parameters themselves (replicated: model.state_dict())."""
    import dataclasses
    hps = getattr(opt, "hps", None) or [opt.hp]
    return {"format": 1, "kind": "adam" if opt.kind == MPO_ADAM else "sgd", "scheme": opt.scheme, "seed": opt.seed,
            "world": opt.world, "rank": opt.rank, "layout": layout_desc, "step_count": int(opt.step_count),
            "resid": opt.resid, "m": opt.m, "v": opt.v, "hp": [dataclasses.asdict(h) for h in hps]}


def _load_shard_state_dict(opt, sd, layout_desc):
    if sd.get("format") != 1:
        raise MpoError(1, "not a sharded residual-optimizer state dict")
    kind = "adam" if opt.kind == MPO_ADAM else "sgd"
    for key, mine in (("kind", kind), ("scheme", opt.scheme), ("world", opt.world), ("rank", opt.rank),
                      ("layout", layout_desc)):
        if sd.get(key) != mine:
            raise MpoError(1, f"state dict {key} {sd.get(key)!r} does not match this optimizer's {mine!r}")
    with torch.no_grad():
        for key in ("resid", "m", "v"):
            src, dst = sd.get(key), getattr(opt, key)
            if (src is None) != (dst is None):
                raise MpoError(1, f"'{key}' present in only one of state dict / optimizer")
            if src is None:
                continue
            if src.dtype != dst.dtype or tuple(src.shape) != tuple(dst.shape):
                raise MpoError(3, f"'{key}' is {src.dtype}{tuple(src.shape)}, expected {dst.dtype}{tuple(dst.shape)}")
            dst.copy_(src)
    opt.step_count = int(sd["step_count"])
    opt.seed = int(sd["seed"])
    hps = getattr(opt, "hps", None) or [opt.hp]
    if len(sd["hp"]) != len(hps):
        raise MpoError(1, "state dict has a different number of hyper-parameter groups")
    for h, d in zip(hps, sd["hp"]):
        for k, v in d.items():
            setattr(h, k, v)


class ShardedResidualOptimizer:
    """Sharded residual-compensated Adam/AdamW (``kind='adam'``) or SGD-momentum (``kind='sgd'``).

    ``params``: CUDA parameters (fp32 -> split into ``fmt``; 16-bit -> residual 0).  They are
    re-pointed at views of one flat value buffer and their ``.grad`` at views of one flat
    gradient buffer, which backward accumulates into.

    ``transport='nccl'`` (default): ``mpo_sharded_step`` (NCCL reduce-scatter -> shard update ->
    NCCL all-gather).  ``transport='p2p'``: value and gradient buffers live in torch symmetric
    memory and one ``mpo_p2p_sharded_step`` kernel per rank reads every rank's gradient shard and
    writes the new values into every rank's replica over NVLink (no collective launches; no
    global-norm clipping).

    The gradients are SUMMED over ranks (R13, R15): pass ``grad_scale = 1 / world`` in the
    hyper-parameters for DistributedDataParallel's mean."""

    def __init__(self, params, kind: str = "adam", fmt: Optional[torch.dtype] = None, group=None,
                 hp=None, exact: bool = True, comm_ptr: Optional[int] = None, scheme: str = "rne",
                 seed: int = 0, transport: str = "nccl", hp_index: Optional[Sequence[int]] = None):
        import torch.distributed as dist
        if transport not in ("nccl", "p2p"):
            raise MpoError(1, "transport must be 'nccl' or 'p2p'")
        self.transport = transport
        self.params = [p for p in params]
        if not self.params:
            raise MpoError(1, "no parameters")
        self.kind = MPO_ADAM if kind == "adam" else MPO_SGD
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.exact = exact
        dev = self.params[0].device
        vdt = fmt if self.params[0].dtype == torch.float32 else self.params[0].dtype
        if vdt not in (torch.float16, torch.bfloat16):
            raise MpoError(3, "fmt must be torch.float16 or torch.bfloat16")
        self.layout = L = ShardLayout([p.numel() for p in self.params], self.world,
                                      align=2 * ALIGN if scheme in ("x8", "x8z") else ALIGN)
        lo, hi = L.shard_range(self.rank)
        # fp32 source of the flat buffer (transient), split once on the device
        src = torch.zeros(L.total, dtype=torch.float32, device=dev)
        for p, o in zip(self.params, L.offsets):
            src[o:o + p.numel()].copy_(p.data.reshape(-1).float())
        self.scheme, self.seed = scheme, int(seed)
        value, resid = api.mpo_split(src, vdt, exact=exact, scheme=scheme, seed=api.step_seed(self.seed, 0),
                                     sr_stream=0)
        if any(p.dtype != torch.float32 for p in self.params):
            # 16-bit params are exactly representable: their residual is zero (P1)
            pass
        del src
        self.resid = resid[lo:hi].clone()
        del resid
        if transport == "p2p":
            # value replica and gradient buffer in symmetric memory: every rank maps every peer's
            # buffers, and mpo_p2p_sharded_step reads / writes them over NVLink
            self.value = _symm_empty(L.total, vdt, dev)
            self.value.copy_(value)
            self.grad = _symm_empty(L.total, vdt, dev)
            self.grad.zero_()
            self._hv = _rendezvous(self.value, group)
            self._hg = _rendezvous(self.grad, group)
            self._vpeers = _peer_addrs(self._hv, self.value, self.rank)
            self._gpeers = _peer_addrs(self._hg, self.grad, self.rank)
        else:
            self.value = value
            self.grad = torch.zeros(L.total, dtype=vdt, device=dev)
        del value
        need_m = self.kind == MPO_ADAM or (hp is not None and getattr(hp, "momentum", 0.0) != 0.0)
        self.m = torch.zeros(L.shard, dtype=torch.float32, device=dev) if need_m else None
        self.v = torch.zeros(L.shard, dtype=torch.float32, device=dev) if self.kind == MPO_ADAM else None
        self.norm_ws = torch.zeros(api.norm_ws_doubles(exact), dtype=torch.float64, device=dev)
        for p, vv, gg in zip(self.params, L.views(self.value, [p.shape for p in self.params]),
                             L.views(self.grad, [p.shape for p in self.params])):
            p.data = vv
            p.grad = gg
        self.hp = hp if hp is not None else (api.AdamParams(lr=1e-3) if self.kind == MPO_ADAM
                                             else api.SgdParams(lr=1e-2))
        # per-parameter hyper-parameter groups (e.g. no weight decay on 1-D tensors): hp is then a
        # list and hp_index names each parameter's group; the shard's pieces form the segment table
        # of mpo_sharded_step_grouped
        self.hps = list(self.hp) if isinstance(self.hp, (list, tuple)) else [self.hp]
        if hp_index is not None and len(hp_index) != len(self.params):
            raise MpoError(1, "hp_index needs one group index per parameter")
        if any(not 0 <= int(h) < len(self.hps) for h in (hp_index or [])):
            raise MpoError(1, "hp_index out of range")
        self.segments = L.segments(self.rank, hp_index) if hp_index is not None else None
        if len(self.hps) > 1 and self.segments is None:
            raise MpoError(1, "several hyper-parameter groups need hp_index")
        self.step_count = 0
        if transport == "p2p" and (getattr(self.hps[0], "max_grad_norm", 0.0) > 0 or len(self.hps) > 1):
            raise MpoError(1, "the P2P fused step has no norm pre-pass and one hyper-parameter group: use "
                              "transport='nccl' for max_grad_norm / hp groups")
        self.comm = None if transport == "p2p" else (comm_ptr if comm_ptr is not None else nccl_comm_ptr(group))

    def zero_grad(self):
        self.grad.zero_()

    @torch.no_grad()
    def step(self):
        self.step_count += 1
        for hp in self.hps:
            if self.kind == MPO_ADAM:
                hp.step = self.step_count
            else:
                hp.first_step = self.step_count == 1
            hp.seed = api.step_seed(self.seed, self.step_count)
        hp = self.hps[0]
        if self.transport == "p2p":
            # every rank's gradients are complete before any rank reads them, and every rank's
            # new values are in place before any rank reads its replica again
            self._hg.barrier(channel=0)
            api.mpo_p2p_sharded_step(self.kind, self.rank, self.world, self._vpeers, self._gpeers, self.resid,
                                     self.m, self.v, self.layout.total, hp, self.value.dtype, exact=self.exact,
                                     scheme=self.scheme)
            self._hv.barrier(channel=0)
            return
        need_ws = getattr(hp, "max_grad_norm", 0.0) > 0 or getattr(hp, "skip_nonfinite", False)
        api.mpo_sharded_step(self.kind, self.comm, self.rank, self.world, self.value, self.grad, self.resid, self.m,
                             self.v, self.hps if self.segments is not None else hp,
                             norm_ws=self.norm_ws if need_ws else None, exact=self.exact, scheme=self.scheme,
                             segments=self.segments)

    def check_comm(self):
        """Raises MpoError(MPO_ENCCL) if the NCCL communicator failed asynchronously (never blocks;
        the sharded step also checks before issuing its collectives)."""
        if self.comm is not None:
            api.mpo_comm_check(self.comm, exact=self.exact)

    def state_dict(self):
        """This rank's shard of the optimizer state (residual / m / v, step count, hyper-parameters);
        every rank saves its own.  Resume needs the same world size, rank and parameter layout."""
        return _shard_state_dict(self, {"sizes": list(self.layout.sizes), "align": self.layout.align})

    def load_state_dict(self, sd):
        _load_shard_state_dict(self, sd, {"sizes": list(self.layout.sizes), "align": self.layout.align})

    def persistent_bytes(self) -> int:
        b = self.value.numel() * 2 + self.grad.numel() * 2 + self.resid.numel() * self.resid.element_size()
        b += 0 if self.m is None else self.m.numel() * 4
        b += 0 if self.v is None else self.v.numel() * 4
        return b


class ShardedResidualAdamW(ShardedResidualOptimizer):
    """SURVEY 8(b)'s `ShardedResidualAdamW(flat_params, process_group, ...)`: the sharded optimizer
    with torch-style Adam/AdamW arguments."""

    def __init__(self, params, process_group=None, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, adamw: bool = True, max_grad_norm: Optional[float] = None,
                 grad_scale: float = 1.0, fmt: Optional[torch.dtype] = None, **kw):
        hp = api.AdamParams(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay, adamw=adamw,
                            max_grad_norm=float(max_grad_norm or 0.0), grad_scale=grad_scale)
        super().__init__(params, kind="adam", fmt=fmt, group=process_group, hp=hp, **kw)


class ShardedResidualSGD(ShardedResidualOptimizer):
    """The sharded optimizer with torch-style SGD(-momentum) arguments."""

    def __init__(self, params, process_group=None, lr: float = 1e-2, momentum: float = 0.0, dampening: float = 0.0,
                 weight_decay: float = 0.0, nesterov: bool = False, grad_scale: float = 1.0,
                 fmt: Optional[torch.dtype] = None, **kw):
        hp = api.SgdParams(lr=lr, momentum=momentum, dampening=dampening, weight_decay=weight_decay, nesterov=nesterov,
                           grad_scale=grad_scale)
        super().__init__(params, kind="sgd", fmt=fmt, group=process_group, hp=hp, **kw)


# ---------------------------------------------------------------------------------------------
# Hook mode x sharding: bucketed reduce-scatter issued from the
# post-accumulate-grad hooks, each bucket's residual-compensated step on this rank's part, and the
# all-gather of its 16-bit values -- overlapped with the rest of backward on a side stream.
# ---------------------------------------------------------------------------------------------
@dataclass
class BucketLayout:
    """Parameters grouped into buckets in backward order (last parameter first); every bucket is
    padded to a multiple of 16*world elements and split into `world` equal contiguous parts, part
    r owned by rank r.  Flat buffers hold the buckets back to back; the rank's state shard is the
    concatenation of its parts."""
    sizes: List[int]
    world: int
    bucket_elems: int = 1 << 22

    def __post_init__(self):
        if self.world < 1:
            raise ValueError("world must be >= 1")
        # 16 elements: every bucket part is 16-byte aligned even for the int8 residual formats
        q = 2 * ALIGN * self.world
        order = list(range(len(self.sizes)))[::-1]          # autograd produces grads roughly in reverse
        self.buckets = []                                    # [(offset, length, [param indices])]
        self.offsets = [0] * len(self.sizes)
        self.bucket_of = [0] * len(self.sizes)
        o = 0
        cur, used = [], 0
        for i in order:
            cur.append(i)
            self.offsets[i] = o + used
            used += (self.sizes[i] + ALIGN - 1) // ALIGN * ALIGN
            if used >= self.bucket_elems:
                length = (used + q - 1) // q * q
                self.buckets.append((o, length, cur))
                o += length
                cur, used = [], 0
        if cur:
            length = (used + q - 1) // q * q
            self.buckets.append((o, length, cur))
            o += length
        for b, (_, _, idx) in enumerate(self.buckets):
            for i in idx:
                self.bucket_of[i] = b
        self.total = o
        self.shard = o // self.world
        # where each bucket's part of this rank starts inside the rank's shard buffers
        self.part_offsets = []
        p = 0
        for _, length, _ in self.buckets:
            self.part_offsets.append(p)
            p += length // self.world

    def views(self, flat: torch.Tensor, shapes: Sequence[torch.Size]):
        return [flat[o:o + n].view(s) for o, n, s in zip(self.offsets, self.sizes, shapes)]

    def global_range_of_part(self, b: int, rank: int):
        o, length, _ = self.buckets[b]
        k = length // self.world
        return o + rank * k, o + (rank + 1) * k


class BucketedShardedOptimizer:
    """Sharded residual Adam/AdamW or SGD-momentum stepped inside backward, bucket by bucket.

    Parameters are re-pointed at views of one flat value buffer and their .grad at views of one
    flat gradient buffer (zeroed after each bucket's reduce-scatter, ready for the next backward).
    When the last gradient of a bucket has been accumulated, its hook records an event on the
    backward's stream and the bucket's ``mpo_sharded_step`` (NCCL reduce-scatter -> update of this
    rank's part -> NCCL all-gather of the 16-bit values) runs on a side stream, overlapping the
    rest of backward.  ``wait()`` (called by the next forward or explicitly) joins the side stream.
    Global-norm clipping is impossible here; the per-bucket found-inf skip is available."""

    def __init__(self, params, kind: str = "adam", fmt: Optional[torch.dtype] = None, group=None, hp=None,
                 bucket_elems: int = 1 << 22, exact: bool = True, comm_ptr: Optional[int] = None,
                 scheme: str = "rne", seed: int = 0):
        import torch.distributed as dist
        self.params = [p for p in params]
        if not self.params:
            raise MpoError(1, "no parameters")
        self.kind = MPO_ADAM if kind == "adam" else MPO_SGD
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.exact, self.scheme, self.seed = exact, scheme, int(seed)
        dev = self.params[0].device
        vdt = fmt if self.params[0].dtype == torch.float32 else self.params[0].dtype
        if vdt not in (torch.float16, torch.bfloat16):
            raise MpoError(3, "fmt must be torch.float16 or torch.bfloat16")
        self.layout = L = BucketLayout([p.numel() for p in self.params], self.world, bucket_elems)
        src = torch.zeros(L.total, dtype=torch.float32, device=dev)
        for p, o in zip(self.params, L.offsets):
            src[o:o + p.numel()].copy_(p.data.reshape(-1).float())
        value, resid_full = api.mpo_split(src, vdt, exact=exact, scheme=scheme, seed=api.step_seed(self.seed, 0),
                                          sr_stream=0)
        del src
        self.value = value
        self.resid = torch.empty(L.shard, dtype=resid_full.dtype, device=dev)
        for b in range(len(L.buckets)):
            lo, hi = L.global_range_of_part(b, self.rank)
            po = L.part_offsets[b]
            self.resid[po:po + hi - lo].copy_(resid_full[lo:hi])
        del resid_full
        self.grad = torch.zeros(L.total, dtype=vdt, device=dev)
        if hp is None:
            hp = api.AdamParams(lr=1e-3) if self.kind == MPO_ADAM else api.SgdParams(lr=1e-2)
        if getattr(hp, "max_grad_norm", 0.0) > 0:
            raise MpoError(1, "global-norm clipping needs every gradient at once: impossible in the fused "
                              "backward (P:93, P:186)")
        self.hp = hp
        need_m = self.kind == MPO_ADAM or getattr(hp, "momentum", 0.0) != 0.0
        self.m = torch.zeros(L.shard, dtype=torch.float32, device=dev) if need_m else None
        self.v = torch.zeros(L.shard, dtype=torch.float32, device=dev) if self.kind == MPO_ADAM else None
        self.norm_ws = torch.zeros(api.norm_ws_doubles(exact), dtype=torch.float64, device=dev)
        shapes = [p.shape for p in self.params]
        for p, vv, gg in zip(self.params, L.views(self.value, shapes), L.views(self.grad, shapes)):
            p.data = vv
            p.grad = gg
        self.comm = comm_ptr if comm_ptr is not None else nccl_comm_ptr(group)
        self.side = torch.cuda.Stream(device=dev)
        self.step_count = 0
        self._pending = [len(idx) for _, _, idx in L.buckets]
        self._handles = [p.register_post_accumulate_grad_hook(self._make_hook(i)) for i, p in enumerate(self.params)]

    def _make_hook(self, i):
        ref = weakref.ref(self)   # hooks live in C++-held tables: no strong cycle back to self

        def hook(p):
            o = ref()
            if o is None:
                return
            b = o.layout.bucket_of[i]
            o._pending[b] -= 1
            if o._pending[b] == 0:
                o._launch_bucket(b)
        return hook

    def _launch_bucket(self, b):
        L = self.layout
        if self._pending.count(0) == 1:        # first bucket of this backward: a new step
            self.step_count += 1
        o, length, _ = L.buckets[b]
        po = L.part_offsets[b]
        k = length // self.world
        hp = self.hp
        if self.kind == MPO_ADAM:
            hp.step = self.step_count
        else:
            hp.first_step = self.step_count == 1
        hp.seed = api.step_seed(self.seed, self.step_count)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.side.wait_event(ev)
        with torch.cuda.stream(self.side):
            # each bucket draws its stochastic-rounding numbers from its own stream (rank + world*b):
            # one shared stream would repeat the same draws in every bucket of a step
            api.mpo_sharded_step(self.kind, self.comm, self.rank, self.world, self.value[o:o + length],
                                 self.grad[o:o + length], self.resid[po:po + k],
                                 None if self.m is None else self.m[po:po + k],
                                 None if self.v is None else self.v[po:po + k], [hp],
                                 norm_ws=self.norm_ws if getattr(hp, "skip_nonfinite", False) else None,
                                 exact=self.exact, scheme=self.scheme, stream=self.side,
                                 segments=[(0, 0, self.rank + self.world * b)])
            self.grad[o:o + length].zero_()       # ready for the next backward's accumulation
        if all(x == 0 for x in self._pending):  # backward done: re-arm the bucket counters
            self._pending = [len(idx) for _, _, idx in L.buckets]

    def state_dict(self):
        """This rank's parts of every bucket's state (see ShardedResidualOptimizer.state_dict)."""
        self.wait()
        return _shard_state_dict(self, {"sizes": list(self.layout.sizes), "bucket_elems": self.layout.bucket_elems})

    def load_state_dict(self, sd):
        self.wait()
        _load_shard_state_dict(self, sd, {"sizes": list(self.layout.sizes), "bucket_elems": self.layout.bucket_elems})

    def wait(self):
        """Make the current stream wait for every bucket step issued so far."""
        torch.cuda.current_stream().wait_stream(self.side)

    def remove_hooks(self):
        for h in self._handles:
            h.remove()
        self._handles = []
