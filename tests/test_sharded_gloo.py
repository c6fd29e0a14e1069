"""The data-parallel sharded path's host logic at world size 2 on CPU (gloo), no GPU.

The GPU path (mpo_sharded_step) is NCCL reduce-scatter -> update of this rank's shard -> NCCL
all-gather of the 16-bit values.  Here the same decomposition is exercised with the product's
ShardLayout and gloo collectives, with the CPU oracle doing the shard update:
* the layout partitions the flat buffer exactly (every element of every parameter in exactly one
  shard; 16-byte-aligned parameter offsets; total a multiple of 8*world);
* sharded == unsharded (P8): per-rank gradients built so the cross-rank sum is exact (reading R13),
  grad_scale = 1/N, then each rank updates only its shard and the all-gathered values equal the
  unsharded oracle step on the mean gradient, bit for bit, for Adam (with and without global-norm
  clipping, whose shard sums are all-reduced) and SGD-momentum.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2309_12381_b200.sharded import ShardLayout

SIZES = [33 * 17, 4096, 5, 128 * 64, 1000, 3]


def test_layout_partitions_exactly():
    for world in (1, 2, 3, 4, 8):
        L = ShardLayout(SIZES, world)
        assert L.total % (8 * world) == 0 and L.shard * world == L.total
        assert all(o % 8 == 0 for o in L.offsets)
        seen = {i: np.zeros(n, np.int32) for i, n in enumerate(SIZES)}
        for r in range(world):
            lo, hi = L.shard_range(r)
            for i, a, b, n in L.owner_slices(r):
                assert 0 <= b and b + n <= L.shard
                assert L.offsets[i] + a == lo + b
                seen[i][a:a + n] += 1
        assert all((c == 1).all() for c in seen.values())
        # params never overlap
        ends = [o + n for o, n in zip(L.offsets, SIZES)]
        assert all(e <= o2 for e, o2 in zip(ends, L.offsets[1:]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_grads(rank, n, fmt):
    # multiples of 2^-12 with |k| <= 16: the 2-rank sum (<= 32 * 2^3 scale, 8 significant bits) and
    # the /2 mean are exact in bf16
    q = synth.rng(77, rank).integers(-16, 17, size=n).astype(np.float32) * np.float32(2.0 ** -12)
    return q


HP_INDEX = [0, 1, 1, 0, 1, 0]          # e.g. decay on matrices only, none on 1-D tensors
GROUP_WD = (0.1, 0.0)


def test_layout_segments():
    """The segment table of mpo_sharded_step_grouped: it partitions each rank's shard from 0, every
    start is a multiple of the alignment (16-B aligned pieces), every parameter piece lies inside
    one segment of its own group, and the stochastic-rounding streams are distinct per rank and
    segment (one segment: stream = rank, like mpo_sharded_step)."""
    for align in (8, 16):
        for world in (1, 2, 3, 8):
            L = ShardLayout(SIZES, world, align=align)
            assert all(o % align == 0 for o in L.offsets) and L.total % (align * world) == 0
            streams = set()
            for r in range(world):
                segs = L.segments(r, HP_INDEX)
                starts = [a for a, _, _ in segs]
                assert starts[0] == 0 and all(a < b for a, b in zip(starts, starts[1:])) and starts[-1] < L.shard
                assert all(a % align == 0 for a in starts)
                ends = starts[1:] + [L.shard]
                for i, _, b, n in L.owner_slices(r):
                    k = max(j for j, a in enumerate(starts) if a <= b)
                    assert b + n <= ends[k] and segs[k][1] == HP_INDEX[i]
                for k, (_, _, st) in enumerate(segs):
                    assert st == r + world * k
                    streams.add(st)
            assert len(streams) == sum(len(L.segments(r, HP_INDEX)) for r in range(world))
            assert L.segments(0, [0] * len(SIZES)) == [(0, 0, 0)]


def _worker(rank, world, port, kind, clip, out_dir, groups=False):
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fmt = "bf16"
        L = ShardLayout(SIZES, world)
        lo, hi = L.shard_range(rank)
        # identical initial flat fp32 weights on every rank, split with the oracle
        w = np.zeros(L.total, np.float32)
        for i, (o, n) in enumerate(zip(L.offsets, SIZES)):
            w[o:o + n] = synth.weights(n, 0.02, 0xB0B + i)
        h, r = oracle.split(fmt, w)
        # this rank's gradient (fp32 exact values) -> 16-bit as the backward would hand it over
        g32 = np.zeros(L.total, np.float32)
        for i, (o, n) in enumerate(zip(L.offsets, SIZES)):
            g32[o:o + n] = _rank_grads(rank, n, fmt)[:n] * np.float32(2.0 ** (i % 4))
        # reduce-scatter (gloo has no reduce_scatter: all_reduce + take the shard; exact sums)
        t = torch.from_numpy(g32.copy())
        dist.all_reduce(t)
        gsum = t.numpy()[lo:hi].copy()
        g16 = synth.to16_bits(gsum, fmt)
        assert np.array_equal(oracle.widen(fmt, g16), gsum)          # the sum is exact in bf16
        hs, rs = h[lo:hi].copy(), r[lo:hi].copy()
        m = np.zeros(L.shard, np.float32)
        v = np.zeros(L.shard, np.float32)
        coef = None
        if kind == "adam" and clip:
            ss = torch.tensor([oracle.sumsq(fmt, g16, 1.0 / world)], dtype=torch.float64)
            dist.all_reduce(ss)
            coef = oracle.clip_coef(float(ss[0]), 0.01)
        if kind == "adam" and groups:
            # per-parameter groups: each segment of the shard with its own hyper-parameters
            segs = L.segments(rank, HP_INDEX)
            ends = [a for a, _, _ in segs[1:]] + [L.shard]
            for (a, hgrp, _), b in zip(segs, ends):
                sl = slice(a, b)
                hh, rr, mm, vv = hs[sl].copy(), rs[sl].copy(), m[sl].copy(), v[sl].copy()
                oracle.adam_step(fmt, fmt, hh, rr, g16[sl].copy(), mm, vv, lr=1e-3, weight_decay=GROUP_WD[hgrp],
                                 grad_scale=1.0 / world, step=1, clip_coef=coef)
                hs[sl], rs[sl] = hh, rr
        elif kind == "adam":
            oracle.adam_step(fmt, fmt, hs, rs, g16, m, v, lr=1e-3, weight_decay=0.1, grad_scale=1.0 / world,
                             step=1, clip_coef=coef)
        else:
            oracle.sgd_step(fmt, fmt, hs, rs, g16, m, lr=0.1, momentum=0.9, grad_scale=1.0 / world, first_step=True)
        # all-gather of the 16-bit values only
        # (gloo has no int16 collectives: the 16-bit patterns travel widened to int32, unchanged)
        parts = [torch.zeros(L.shard, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(hs.astype(np.int32)))
        value = torch.cat(parts).numpy().astype(np.uint16)
        np.save(os.path.join(out_dir, f"value_{rank}.npy"), value)
        np.save(os.path.join(out_dir, f"resid_{rank}.npy"), rs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,clip,groups", [("adam", False, False), ("adam", True, False), ("sgd", False, False),
                                              ("adam", True, True)])
def test_sharded_equals_unsharded_world2(tmp_path, orc, kind, clip, groups):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), kind, clip, str(tmp_path), groups), nprocs=world, join=True)
    fmt = "bf16"
    L = ShardLayout(SIZES, world)
    w = np.zeros(L.total, np.float32)
    g = np.zeros(L.total, np.float32)
    for i, (o, n) in enumerate(zip(L.offsets, SIZES)):
        w[o:o + n] = synth.weights(n, 0.02, 0xB0B + i)
        g[o:o + n] = sum(_rank_grads(rk, n, fmt) for rk in range(world)) * np.float32(2.0 ** (i % 4))
    h, r = orc.split(fmt, w)
    g16 = synth.to16_bits(g, fmt)
    m = np.zeros(L.total, np.float32)
    v = np.zeros(L.total, np.float32)
    if kind == "adam":
        coef = orc.clip_coef(orc.sumsq(fmt, g16, 1.0 / world), 0.01) if clip else None
        if clip:
            assert coef < 1.0
        if groups:   # unsharded reference: every parameter stepped with its own group
            for i, (o, n) in enumerate(zip(L.offsets, SIZES)):
                sl = slice(o, o + n)
                hh, rr, mm, vv = h[sl].copy(), r[sl].copy(), m[sl].copy(), v[sl].copy()
                orc.adam_step(fmt, fmt, hh, rr, g16[sl].copy(), mm, vv, lr=1e-3, weight_decay=GROUP_WD[HP_INDEX[i]],
                              grad_scale=1.0 / world, step=1, clip_coef=coef)
                h[sl], r[sl] = hh, rr
        else:
            orc.adam_step(fmt, fmt, h, r, g16, m, v, lr=1e-3, weight_decay=0.1, grad_scale=1.0 / world, step=1,
                          clip_coef=coef)
    else:
        orc.sgd_step(fmt, fmt, h, r, g16, m, lr=0.1, momentum=0.9, grad_scale=1.0 / world, first_step=True)
    for rank in range(world):
        assert np.array_equal(np.load(tmp_path / f"value_{rank}.npy"), h)
        lo, hi = L.shard_range(rank)
        assert np.array_equal(np.load(tmp_path / f"resid_{rank}.npy"), r[lo:hi])


def test_bucket_layout_partitions_exactly():
    from paper_2309_12381_b200.sharded import BucketLayout
    for world in (1, 2, 4, 8):
        for be in (64, 4096, 1 << 20):
            L = BucketLayout(SIZES, world, be)
            assert L.total % (16 * world) == 0 and L.shard * world == L.total
            seen = sorted(i for _, _, idx in L.buckets for i in idx)
            assert seen == list(range(len(SIZES)))                         # every param in one bucket
            for b, (o, length, idx) in enumerate(L.buckets):
                assert o % 16 == 0 and length % (16 * world) == 0
                for i in idx:                                              # params inside their bucket
                    assert o <= L.offsets[i] and L.offsets[i] + SIZES[i] <= o + length
                    assert L.offsets[i] % 8 == 0
                parts = [L.global_range_of_part(b, r) for r in range(world)]
                assert parts[0][0] == o and parts[-1][1] == o + length
                assert all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))
                assert L.part_offsets[b] % 16 == 0
            spans = sorted((L.offsets[i], L.offsets[i] + n) for i, n in enumerate(SIZES))
            assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))   # no overlap
