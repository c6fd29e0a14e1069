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

    def __post_init__(self):
        if self.world < 1:
            raise ValueError("world must be >= 1")
        offs, o = [], 0
        for n in self.sizes:
            offs.append(o)
            o += (n + ALIGN - 1) // ALIGN * ALIGN
        q = ALIGN * self.world
        self.offsets = offs
        self.used = o
        self.total = (o + q - 1) // q * q
        self.shard = self.total // self.world

    def shard_range(self, rank: int):
        return rank * self.shard, (rank + 1) * self.shard

    def views(self, flat: torch.Tensor, shapes: Sequence[torch.Size]):
        return [flat[o:o + n].view(s) for o, n, s in zip(self.offsets, self.sizes, shapes)]

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


class ShardedResidualOptimizer:
    """Sharded residual-compensated Adam/AdamW (``kind='adam'``) or SGD-momentum (``kind='sgd'``).

    ``params``: CUDA parameters (fp32 -> split into ``fmt``; 16-bit -> residual 0).  They are
    re-pointed at views of one flat value buffer and their ``.grad`` at views of one flat
    gradient buffer, which backward accumulates into."""

    def __init__(self, params, kind: str = "adam", fmt: Optional[torch.dtype] = None, group=None,
                 hp=None, exact: bool = False, comm_ptr: Optional[int] = None, scheme: str = "rne",
                 seed: int = 0):
        import torch.distributed as dist
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
        self.layout = L = ShardLayout([p.numel() for p in self.params], self.world)
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
        self.value = value
        self.resid = resid[lo:hi].clone()
        del resid
        self.grad = torch.zeros(L.total, dtype=vdt, device=dev)
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
        self.step_count = 0
        self.comm = comm_ptr if comm_ptr is not None else nccl_comm_ptr(group)

    def zero_grad(self):
        self.grad.zero_()

    @torch.no_grad()
    def step(self):
        self.step_count += 1
        hp = self.hp
        if self.kind == MPO_ADAM:
            hp.step = self.step_count
        else:
            hp.first_step = self.step_count == 1
        hp.seed = api.step_seed(self.seed, self.step_count)
        api.mpo_sharded_step(self.kind, self.comm, self.rank, self.world, self.value, self.grad, self.resid, self.m,
                             self.v, hp, norm_ws=self.norm_ws if getattr(hp, "max_grad_norm", 0.0) > 0 else None,
                             exact=self.exact, scheme=self.scheme)

    def persistent_bytes(self) -> int:
        b = self.value.numel() * 2 + self.grad.numel() * 2 + self.resid.numel() * self.resid.element_size()
        b += 0 if self.m is None else self.m.numel() * 4
        b += 0 if self.v is None else self.v.numel() * 4
        return b
