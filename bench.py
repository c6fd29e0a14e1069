#!/usr/bin/env python
"""bench.py -- optimizer-step throughput of the residual-compensated 16-bit step on B200.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mpo|reference] [--workload NAME]
prints ONE JSON line on rank 0.

* A "step" is one pass of the whole hot path over the workload's parameter set: reconstruct ->
  update -> re-split for every parameter, in one multi-tensor launch; at N>1
  the data-parallel sharded step (NCCL reduce-scatter of 16-bit grads -> shard update -> NCCL
  all-gather of 16-bit values).
* Default workload = BASELINE.json configs[3], the largest single-GPU configuration and the Adam
  step BASELINE.json's target names: the LLaMA-7B parameter set (6 738 415 616 params, 291
  tensors), bf16 + int16 residual, Adam (lr 3e-4, betas (0.9, 0.95), eps 1e-8), one multi-tensor
  launch per step at N=1 (175 GB of algorithmic traffic per step >> 126 MB L2: no flush needed);
  at N>1 the sharded step.
* value = params/s over all ranks (device time, CUDA events, max over ranks).
* Secondary (N=1): ResNet-50 SGD-momentum (configs[1]), GPT-2 small AdamW (configs[2] parameter
  set), ViT-L/16 Adam + global-norm clip (configs[4]), the flat 2^20 Adam tensor (configs[0]:
  launch/L2-bound and L2-flushed), the storage variants, and the GPT-2 hook-mode training step --
  each with its own roofline fraction or breakdown.
* cpu_baseline: the CPU oracle (oracle/, plain C) on a bounded sample, single-threaded AND with
  its OpenMP build over every core of the affinity mask (bit-identical builds).
* --impl reference: the CPU oracle (OpenMP build, all cores) on a bounded sample of the same
  workload: the reference arm of this tier (there is no reference code to install).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
WORKLOADS = {
    # name: (synth workload, value fmt, optimizer, hyper-parameters, BASELINE config index)
    "resnet50_sgd": ("resnet50", "fp16", "sgd", dict(lr=0.3, momentum=0.9, weight_decay=2e-4), 1),
    # plain SGD (no momentum buffer): the 10 B/param row of SURVEY 8(a)'s byte table
    "resnet50_sgd_plain": ("resnet50", "fp16", "sgd", dict(lr=0.3, momentum=0.0, weight_decay=2e-4), 1),
    "gpt2_adamw": ("gpt2_small", "bf16", "adam", dict(lr=6e-4, beta1=0.9, beta2=0.95, eps=1e-8,
                                                      weight_decay=0.1, adamw=True), 2),
    "vit_l16_adam_clip": ("vit_l16", "fp16", "adam", dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8,
                                                         max_grad_norm=1.0, adamw=False), 4),
    "llama7b_adam": ("llama7b", "bf16", "adam", dict(lr=3e-4, beta1=0.9, beta2=0.95, eps=1e-8, adamw=False), 3),
    "flat1m_adam": ("flat1m", "fp16", "adam", dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, adamw=False), 0),
}
DEFAULT_WORKLOAD = "llama7b_adam"
# algorithmic HBM bytes per parameter per step
BYTES_PER_PARAM = {"sgd": 18, "adam": 26, "adam_clip": 28}


def workload_config(name):
    """The bench line's `config` (identical in both arms): the workload and its hyper-parameters."""
    from synth import workloads
    wl, fmt, kind, hp, cfg = WORKLOADS[name]
    sizes = workloads.sizes(wl)
    return {"workload": f"{name}: BASELINE configs[{cfg}] parameter set {wl} ({sum(sizes)} params, "
                        f"{len(sizes)} tensors)",
            "optimizer": kind, "hyper_parameters": hp, "value_dtype": fmt}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def same_box_copy_gbs():
    """The copy bandwidth of THIS box, measured like MEASURED_PEAKS.json's hbm_gbs (torch copy of
    1 Gi bf16 elements, read + write bytes, best of 10, CUDA events): boxes differ by a few %, so the
    line also states the kernel's fraction of its own box's copy (the roofline peak stays the
    driver-measured number)."""
    import torch
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    best = None
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    del a, b
    torch.cuda.empty_cache()
    return 2 * 2 * (1 << 30) / (best * 1e-3) / 1e9


def ncu_traffic(workload):
    """dram read+write bytes per launch of the step kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
# clocks during the timed region
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.windows = []
        # nvidia-smi takes a moment to start: wait (<= 5 s) for its first sample, so that even a
        # timed region shorter than that has samples before and after it
        t_end = time.time() + 5.0
        while self.p is not None and time.time() < t_end:
            self.f.flush()
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.02)

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [l.strip().split(", ") for l in open(self.f.name) if l.strip()]
        os.unlink(self.f.name)
        sel = []
        for r in rows:
            try:
                ts = time.mktime(time.strptime(r[0].split(".")[0], "%Y/%m/%d %H:%M:%S")) + float("0." + r[0].split(".")[1])
            except Exception:
                continue
            if any(a - 0.1 <= ts <= b + 0.1 for a, b in self.windows):
                sel.append(r)
        if not sel and rows and self.windows:
            # a region shorter than the sampling period: the samples just before and after it
            a, b = self.windows[0][0], self.windows[-1][1]
            ts = []
            for r in rows:
                try:
                    ts.append(time.mktime(time.strptime(r[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                              + float("0." + r[0].split(".")[1]))
                except Exception:
                    ts.append(None)
            before = [r for r, t in zip(rows, ts) if t is not None and t <= a]
            after = [r for r, t in zip(rows, ts) if t is not None and t >= b]
            sel = before[-1:] + after[:1]
        use = sel if sel else rows
        sm = [float(r[1]) for r in use if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in use if r[2].replace(".", "").isdigit()]
        reasons = sorted({n for r in use for n, v in zip(self.NAMES, r[3:7]) if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sel), "samples_total": len(rows)}


# ------------------------------------------------------------------------------------------
# device-side state for one workload
# ------------------------------------------------------------------------------------------
class Workload:
    """Flat value / residual / grad / state buffers with one 16-B aligned view per parameter
    (ShardLayout), and the cached multi-tensor table."""

    def __init__(self, name, world=1, rank=0, seed=0xB0B, scheme="rne"):
        import torch
        import paper_2309_12381_b200 as mpo
        from synth import torch_normal_, workloads
        self.name = name
        self.scheme = scheme
        wl, fmt, kind, hp, cfg = WORKLOADS[name]
        self.kind, self.fmt, self.hpkw, self.cfg = kind, fmt, hp, cfg
        self.sizes = workloads.sizes(wl)
        self.P = sum(self.sizes)
        self.ntensors = len(self.sizes)
        self.tdt = torch.float16 if fmt == "fp16" else torch.bfloat16
        self.world, self.rank = world, rank
        dev = torch.device("cuda")
        self.layout = mpo.ShardLayout(self.sizes, world)
        L = self.layout
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        self.value = torch.empty(L.total, dtype=self.tdt, device=dev)
        # fp32 init, split on the device chunk by chunk (N(0,0.02), seeded)
        rdt = mpo.api.resid_dtype(scheme)
        resid_full = torch.empty(L.shard if world > 1 else L.total, dtype=rdt, device=dev)
        chunk = 1 << 28
        lo, hi = L.shard_range(rank) if world > 1 else (0, L.total)
        tmp_r = torch.empty(min(chunk, L.total), dtype=rdt, device=dev)
        for s in range(0, L.total, chunk):
            e = min(L.total, s + chunk)
            w32 = torch.empty(e - s, dtype=torch.float32, device=dev)
            torch_normal_(w32, 0.02, seed, s // chunk)
            mpo.mpo_split(w32, self.tdt, value=self.value[s:e], resid=tmp_r[:e - s], scheme=scheme, seed=seed,
                          sr_stream=s // chunk)
            a, b = max(s, lo), min(e, hi)
            if a < b:
                resid_full[a - lo:b - lo].copy_(tmp_r[a - s:b - s])
            del w32
        del tmp_r
        self.resid = resid_full
        self.grad = torch.empty(L.total, dtype=self.tdt, device=dev)
        torch_normal_(self.grad, 1e-3 if kind == "adam" else 1e-2, seed, 1000 + rank)
        if kind == "adam" and "max_grad_norm" in hp:
            # scale so the global norm is ~4 (clipping active)
            self.grad.mul_(4.0 / math.sqrt(self.P) / 1e-3)
        n_state = L.shard if world > 1 else L.total
        plain_sgd = kind == "sgd" and not hp.get("momentum", 0.0)
        self.m = None if plain_sgd else torch.zeros(n_state, dtype=torch.float32, device=dev)
        self.v = torch.zeros(n_state, dtype=torch.float32, device=dev) if kind == "adam" else None
        self.norm_ws = torch.zeros(mpo.norm_ws_doubles(), dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        self.persistent_bytes = torch.cuda.memory_allocated() - base
        self.t = 0
        self.mpo = mpo
        if world == 1:
            shapes = [(n,) for n in self.sizes]
            V = L.views(self.value, shapes)
            R = L.views(self.resid, shapes)
            G = L.views(self.grad, shapes)
            M = L.views(self.m, shapes) if self.m is not None else [None] * len(shapes)
            W = L.views(self.v, shapes) if self.v is not None else [None] * len(shapes)
            self.table = mpo.TensorTable(V, R, G, M, W, scheme=scheme)
        self.comm = None

    def release(self):
        """Drop the device buffers (host-side attributes stay for reporting)."""
        import torch
        self.value = self.resid = self.grad = self.m = self.v = self.table = None
        torch.cuda.empty_cache()

    @property
    def clip(self):
        return self.kind == "adam" and self.hpkw.get("max_grad_norm", 0.0) > 0

    @property
    def bytes_per_param(self):
        b = BYTES_PER_PARAM["adam_clip" if self.clip else self.kind]
        if self.kind == "sgd" and not self.hpkw.get("momentum", 0.0):
            b = 10                                    # value + residual + grad in, value + residual out
        return b - 2 if self.scheme in ("x8", "x8z") else b      # 8-bit residual: 1 B read + 1 B written

    def hp(self):
        mpo = self.mpo
        seed = mpo.api.step_seed(0xB0B, self.t)
        if self.kind == "sgd":
            return mpo.SgdParams(first_step=(self.t == 1), seed=seed, **self.hpkw)
        return mpo.AdamParams(step=self.t, seed=seed, **self.hpkw)

    def step(self, sharded=False):
        """One pass of the hot path (one C-ABI call)."""
        self.t += 1
        mpo = self.mpo
        hp = self.hp()
        if sharded or self.world > 1:
            from paper_2309_12381_b200._lib import MPO_ADAM, MPO_SGD
            if self.comm is None:
                import torch.distributed as tdist
                from paper_2309_12381_b200.sharded import nccl_comm_ptr
                if not tdist.is_initialized():   # world 1: a single-rank NCCL group (no-op RS/AG)
                    _single_rank_group()
                self.comm = nccl_comm_ptr()
            mpo.mpo_sharded_step(MPO_ADAM if self.kind == "adam" else MPO_SGD, self.comm, self.rank, self.world,
                                 self.value, self.grad, self.resid, self.m, self.v, hp,
                                 norm_ws=self.norm_ws if self.clip else None, scheme=self.scheme)
        elif self.kind == "sgd":
            mpo.mpo_sgd_step(self.table, hp)
        else:
            mpo.mpo_adam_step(self.table, hp, norm_ws=self.norm_ws if self.clip else None)


def timed(fn, steps, warmup, dist=None, sampler=None):
    """W untimed warm-up steps; then K steps bracketed by barrier + synchronize, timed with two CUDA
    events on the current (launching) stream around the whole region (per-step events would add
    ~7 us of gaps per step on a 90 us kernel).  Returns (ms_per_step max over ranks, launches of
    this library inside the region)."""
    import torch
    from paper_2309_12381_b200 import api
    tw = time.time()
    for _ in range(warmup):
        fn()
    s = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = api.launch_count()
    t0 = time.time()
    start.record(s)
    for _ in range(steps):
        fn()
    end.record(s)
    torch.cuda.synchronize()
    t1 = time.time()
    if dist is not None:
        dist.barrier()
    if sampler is not None:
        # the clocks of the warm-up count too: at 20 steps the timed region alone can be shorter
        # than nvidia-smi's sampling period
        sampler.mark(tw, t1)
    launches = api.launch_count() - n0
    ms = start.elapsed_time(end) / steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    return ms, launches


NVLINK_GBS = 900.0   # NVLink 5 per direction per GPU


def multi_gpu_breakdown(wl, dist, steps, warmup, p2p=False):
    """N > 1 only (every rank runs it; collectives in the same order on all ranks).  SURVEY 8(e):
    (i) the update alone on this rank's shard (same step kernel through mpo_sgd_step /
    mpo_adam_step on a one-tensor table of the shard), aggregate params/s = P / max-rank time --
    the part that should scale ~linearly in N; (ii) the two collectives of the sharded step alone
    (NCCL reduce-scatter of the 16-bit grads, all-gather of the 16-bit values, torch's process
    group, same byte counts), as algbw and busbw = bytes*(N-1)/N / t against NVLink's 900 GB/s."""
    import torch
    mpo = wl.mpo
    L, N = wl.layout, wl.world
    lo, hi = L.shard_range(wl.rank)
    tab = mpo.TensorTable([wl.value[lo:hi]], [wl.resid], [wl.grad[lo:hi]], [wl.m],
                          [wl.v if wl.v is not None else None], scheme=wl.scheme)

    def upd():
        wl.t += 1
        if wl.kind == "sgd":
            mpo.mpo_sgd_step(tab, wl.hp())
        else:
            mpo.mpo_adam_step(tab, wl.hp(), norm_ws=wl.norm_ws if wl.clip else None)

    out = {}
    t_upd, _ = timed(upd, steps, warmup, dist)
    out["update_only"] = {"ms_per_step": t_upd, "params_per_s": wl.P / (t_upd * 1e-3),
                          "shard_params": hi - lo,
                          "achieved_gbs_per_rank": (hi - lo) * wl.bytes_per_param / (t_upd * 1e-3) / 1e9}
    rs_out = torch.empty(hi - lo, dtype=wl.grad.dtype, device=wl.grad.device)
    ag_out = torch.empty_like(wl.value)
    nbytes = wl.value.numel() * wl.value.element_size()
    for name, fn in (("reduce_scatter_grad16", lambda: dist.reduce_scatter_tensor(rs_out, wl.grad)),
                     ("all_gather_value16", lambda: dist.all_gather_into_tensor(ag_out, wl.value[lo:hi]))):
        ms, _ = timed(fn, max(10, steps // 10), warmup, dist)
        algbw = nbytes / (ms * 1e-3) / 1e9
        busbw = algbw * (N - 1) / N
        out[name] = {"ms": ms, "bytes": nbytes, "algbw_gbs": algbw, "busbw_gbs": busbw,
                     "frac_of_nvlink_900": busbw / NVLINK_GBS}
    del rs_out, ag_out
    out["nccl_algo"] = os.environ.get("NCCL_ALGO", "auto (NCCL's choice; NCCL_DEBUG=INFO names it)")
    # the same step fused with its collectives over NVLink peer memory (mpo_p2p_sharded_step on
    # torch symmetric memory, between symmetric-memory barriers) and over NVLS multicast, when the
    # box provides them.  A symmetric-memory rendezvous that failed on some ranks only would hang
    # the others, so every rank first checks what it can do locally (symmetric memory importable,
    # peer access to every other local GPU) and the ranks agree (all_reduce MIN) before any
    # rendezvous; --no-p2p skips it altogether
    if p2p and not wl.clip:
        ok = 1
        try:
            import torch.distributed._symmetric_memory  # noqa: F401
            me = torch.cuda.current_device()
            ok = int(all(torch.cuda.can_device_access_peer(me, j) for j in range(torch.cuda.device_count())
                         if j != me))
        except Exception:
            ok = 0
        t = torch.tensor([ok], device="cuda", dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if not int(t.item()):
            out["p2p_fused_step"] = {"skipped": "no symmetric memory / peer access on every rank"}
        elif N > 1 or os.environ.get("MPO_BENCH_FUSED_CHILD") == "1":   # (the env: exercise it at N=1)
            # in child processes (one per rank, their own process group): a device fault in a fused
            # kernel on hardware this code has never run on then costs the child, not this line
            out.update(_fused_in_children(wl, steps, warmup))
        else:
            try:
                out.update(_p2p_fused_timing(wl, dist, steps, warmup))
            except Exception as ex:
                out["p2p_fused_step"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    return out


def _fused_in_children(wl, steps, warmup, timeout_s=300):
    """Every rank runs `bench.py --fused-child` (same workload, a fresh process group on
    MASTER_PORT + 101) and reads its JSON line; an error or a timeout is reported, not raised."""
    import torch
    torch.cuda.empty_cache()                 # the children need the memory this process cached
    env = dict(os.environ)
    env["MASTER_PORT"] = str(int(os.environ.get("MASTER_PORT", "29500")) + 101)
    env.pop("TORCHELASTIC_USE_AGENT_STORE", None)   # the child group hosts its own store
    cmd = [sys.executable, os.path.abspath(__file__), "--fused-child", "--workload", wl.name, "--steps", str(steps),
           "--warmup", str(warmup)]
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout_s)
        lines = [line for line in r.stdout.splitlines() if line.startswith("{")]
        if lines:
            return json.loads(lines[-1])
        return {"p2p_fused_step": {"error": f"child rc={r.returncode}: {r.stderr[-300:]}"}}
    except subprocess.TimeoutExpired:
        return {"p2p_fused_step": {"error": f"child timed out after {timeout_s} s"}}


def fused_child(args):
    """--fused-child (started by _fused_in_children on every rank): the P2P and NVLS fused sharded
    steps on this workload, one JSON line with their timings."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{local}"))
    try:
        wl = Workload(args.workload, world, rank)
        res = _p2p_fused_timing(wl, dist, args.steps, args.warmup)
    except Exception as ex:
        res = {"p2p_fused_step": {"error": f"{type(ex).__name__}: {ex}"[:300]}}
    emit(res)
    dist.destroy_process_group()


def _p2p_fused_timing(wl, dist, steps, warmup):
    from paper_2309_12381_b200 import api
    from paper_2309_12381_b200._lib import MPO_ADAM, MPO_SGD
    from paper_2309_12381_b200.sharded import _peer_addrs, _rendezvous, _symm_empty
    L, N, r = wl.layout, wl.world, wl.rank
    val = _symm_empty(L.total, wl.value.dtype, wl.value.device)
    grd = _symm_empty(L.total, wl.grad.dtype, wl.grad.device)
    val.copy_(wl.value)
    grd.copy_(wl.grad)
    hv, hg = _rendezvous(val, None), _rendezvous(grd, None)
    vp, gp = _peer_addrs(hv, val, r), _peer_addrs(hg, grd, r)
    kind = MPO_ADAM if wl.kind == "adam" else MPO_SGD

    def step():
        wl.t += 1
        hg.barrier(channel=0)
        api.mpo_p2p_sharded_step(kind, r, N, vp, gp, wl.resid, wl.m, wl.v, L.total, wl.hp(), wl.value.dtype,
                                 scheme=wl.scheme)
        hv.barrier(channel=0)

    ms, launches = timed(step, steps, warmup, dist)
    res = {"p2p_fused_step": {
        "ms_per_step": ms, "params_per_s": wl.P / (ms * 1e-3), "launches_per_step": launches / steps,
        "nvlink_bytes_per_rank_per_step": 2 * 2 * L.shard * (N - 1),
        "nvlink_gbs_per_rank": 2 * 2 * L.shard * (N - 1) / (ms * 1e-3) / 1e9,
        "note": "one kernel per rank: bulk copies of every rank's grad shard (fp32 sum in rank order), update, "
                "P2P stores of the new values into every replica; + 2 symmetric-memory barriers"}}
    # NVLS: the same buffers' multicast object, when every rank has one (all ranks agree first)
    import torch
    mc_v, mc_g = int(getattr(hv, "multicast_ptr", 0) or 0), int(getattr(hg, "multicast_ptr", 0) or 0)
    t = torch.tensor([1 if (mc_v and mc_g and wl.scheme == "rne") else 0], device="cuda", dtype=torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if int(t.item()):
        off_v, off_g = val.data_ptr() - int(hv.buffer_ptrs[r]), grd.data_ptr() - int(hg.buffer_ptrs[r])
        vdt = api.format_code(wl.value.dtype)

        def nvls():
            wl.t += 1
            hg.barrier(channel=0)
            api.mpo_nvls_sharded_step(kind, r, N, vdt, mc_v + off_v, val.data_ptr(), mc_g + off_g, wl.resid, wl.m,
                                      wl.v, L.total, wl.hp())
            hv.barrier(channel=0)
        try:
            ms2, l2 = timed(nvls, steps, warmup, dist)
            res["nvls_fused_step"] = {"ms_per_step": ms2, "params_per_s": wl.P / (ms2 * 1e-3),
                                      "launches_per_step": l2 / steps,
                                      "note": "multimem.ld_reduce of the grad shard (fp32 in-switch sum), update, "
                                              "multimem.st of the values; + 2 symmetric-memory barriers"}
        except Exception as ex:
            res["nvls_fused_step"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    else:
        res["nvls_fused_step"] = {"skipped": "no multicast object on every rank (or a non-RNE scheme)"}
    del val, grd
    return res


def e2e_measure(wl, steps, dist=None):
    """Same metric end to end through the public optimizer API with host buffers: every step copies
    the step's 16-bit gradients host(pinned)->device, runs ResidualSGD/ResidualAdamW.step(), and
    reads the updated 16-bit values device->host."""
    import torch
    import paper_2309_12381_b200 as mpo
    from synth import torch_normal_
    sizes = wl.sizes if wl.world == 1 else None
    dev = torch.device("cuda")
    if wl.world == 1:
        # Parameters are views of one flat value buffer; gradients are views of one of two flat
        # device buffers (double-buffered).  Per step: H2D of the step's grads on a copy-in stream
        # (overlapping the previous step), ResidualSGD/ResidualAdamW.step() on the compute stream,
        # a device copy of the updated values into a staging buffer, and the D2H of that staging
        # buffer on a copy-out stream (overlapping the next step).  PCIe's two directions run
        # concurrently; every byte still crosses inside the timed region.
        L = wl.layout
        flat_v = torch.empty(L.total, dtype=wl.tdt, device=dev)
        torch_normal_(flat_v, 0.02, 0xB0B, 5000)
        gbuf = [torch.zeros(L.total, dtype=wl.tdt, device=dev) for _ in range(2)]
        stage = [torch.empty(L.total, dtype=wl.tdt, device=dev) for _ in range(2)]
        shapes = [(n,) for n in sizes]
        params = [torch.nn.Parameter(v) for v in L.views(flat_v, shapes)]
        gviews = [L.views(g, shapes) for g in gbuf]
        for p, g in zip(params, gviews[0]):
            p.grad = g
        hk = dict(wl.hpkw)
        b1b2 = (hk.pop("beta1"), hk.pop("beta2")) if wl.kind != "sgd" else None
        # the step is cut into C chunks of parameters (one optimizer each, ~equal bytes) so that the
        # D2H of a chunk's new values starts as soon as that chunk is stepped and the H2D of the next
        # step's chunk as soon as this step consumed it: both PCIe directions stay busy and the
        # compute hides under them (one optimizer over everything: the 29 ms LLaMA step sat between
        # the two transfers on the critical path, 315 ms/step vs a ~280 ms PCIe bound)
        C = 8 if len(params) >= 16 else 1
        target = L.total / C
        bounds, acc = [0], 0
        for i, n_ in enumerate(sizes):
            acc += n_
            if acc >= target * len(bounds) and len(bounds) < C:
                bounds.append(i + 1)
        bounds.append(len(params))
        chunks = [(a_, b_) for a_, b_ in zip(bounds[:-1], bounds[1:]) if b_ > a_]
        ranges = [(L.offsets[a_], L.offsets[b_] if b_ < len(params) else L.total) for a_, b_ in chunks]
        opts = []
        for a_, b_ in chunks:
            ps = params[a_:b_]
            opts.append(mpo.ResidualSGD(ps, **hk) if wl.kind == "sgd" else mpo.ResidualAdamW(ps, betas=b1b2, **hk))
        host = [torch.empty(L.total, dtype=wl.tdt, pin_memory=True) for _ in range(2)]
        sig = 1e-3 if wl.kind == "adam" else 1e-2
        for k, h in enumerate(host):
            # real gradients: seeded N(0, sigma) cast to the value dtype (finite, the bench's own scale);
            # drawn on the device once, before any timing, then kept in pinned host memory
            torch_normal_(gbuf[k], sig, 0xB0B, 7000 + k)
            h.copy_(gbuf[k])
        out = torch.empty(L.total, dtype=wl.tdt, pin_memory=True)
        comp = torch.cuda.current_stream()
        cin, cout = torch.cuda.Stream(), torch.cuda.Stream()
        nC = len(chunks)
        state = {"i": 0, "in_ev": [[None] * nC, [None] * nC], "used_ev": [[None] * nC, [None] * nC],
                 "out_ev": [[None] * nC, [None] * nC]}

        def issue_h2d(k, c):
            lo, hi = ranges[c]
            with torch.cuda.stream(cin):
                if state["used_ev"][k][c] is not None:
                    cin.wait_event(state["used_ev"][k][c])    # the step that last read this slice is done
                gbuf[k][lo:hi].copy_(host[k][lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cin)
                state["in_ev"][k][c] = ev

        def step():
            i = state["i"]
            k = i % 2
            for c, ((a_, b_), (lo, hi), opt) in enumerate(zip(chunks, ranges, opts)):
                if state["in_ev"][k][c] is None:
                    issue_h2d(k, c)
                comp.wait_event(state["in_ev"][k][c])
                for p, g in zip(params[a_:b_], gviews[k][a_:b_]):
                    p.grad = g
                opt.step()
                ev = torch.cuda.Event()
                ev.record(comp)
                state["used_ev"][k][c] = ev
                if state["out_ev"][k][c] is not None:
                    comp.wait_event(state["out_ev"][k][c])    # staging slice drained to host
                stage[k][lo:hi].copy_(flat_v[lo:hi])
                done = torch.cuda.Event()
                done.record(comp)
                with torch.cuda.stream(cout):
                    cout.wait_event(done)
                    out[lo:hi].copy_(stage[k][lo:hi], non_blocking=True)
                    oe = torch.cuda.Event()
                    oe.record(cout)
                    state["out_ev"][k][c] = oe
                state["in_ev"][k][c] = None
                if i + 1 != state.get("last", -1):
                    issue_h2d(1 - k, c)                       # prefetch the next step's slice
            state["i"] = i + 1

        def drain():
            comp.wait_stream(cout)
            comp.wait_stream(cin)
        h2d = d2h = L.total * 2
    else:
        # data parallel: every rank's backward hands over its full 16-bit gradient (H2D of all of it)
        # and the step's result is this rank's shard of the new values (D2H of 1/N; after the
        # all-gather every replica holds the same values).  Pinned host memory per rank: grads + shard.
        L = wl.layout
        lo, hi = L.shard_range(wl.rank)
        need = (L.total + (hi - lo)) * 2 * int(os.environ.get("LOCAL_WORLD_SIZE", wl.world))
        avail = _mem_available()
        ok = torch.tensor([0 if (avail is not None and need > 0.7 * avail) else 1], device=dev, dtype=torch.int32)
        if dist is not None:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)      # every rank measures or none does
        if not int(ok.item()):
            return {"skipped": f"host memory: {need / 1e9:.0f} GB of pinned buffers over the local ranks > 70 % "
                               f"of MemAvailable {(avail or 0) / 1e9:.0f} GB on some rank"}
        host = torch.empty(L.total, dtype=wl.tdt, pin_memory=True)
        tmp = torch.empty(L.total, dtype=wl.tdt, device=dev)
        torch_normal_(tmp, 1e-3 if wl.kind == "adam" else 1e-2, 0xB0B, 7000 + wl.rank)
        host.copy_(tmp)
        del tmp
        out = torch.empty(hi - lo, dtype=wl.tdt, pin_memory=True)

        def step():
            wl.grad.copy_(host, non_blocking=True)
            wl.step()
            out.copy_(wl.value[lo:hi], non_blocking=True)
        h2d, d2h = L.total * 2, (hi - lo) * 2
    if wl.world == 1:
        def step_and_drain():
            step()
            if state["i"] == state_target[0]:
                drain()                      # the last timed step's D2H lands inside the region
        state_target = [0]
        for _ in range(3):
            step()
        drain()
        torch.cuda.synchronize()
        state["in_ev"] = [[None] * nC, [None] * nC]   # the first timed step issues its own H2D inside the region
        state_target[0] = state["i"] + steps
        state["last"] = state_target[0]                 # ... and the last one prefetches nothing
        ms, _ = timed(step_and_drain, steps, 0, dist)
    else:
        ms, _ = timed(step, steps, 3, dist)
    # the step really updated finite weights (no special-value slow path was timed)
    finite = bool(torch.isfinite(flat_v if wl.world == 1 else wl.value).all().item())
    if not finite:
        raise RuntimeError("e2e: non-finite weights after the timed steps")
    return {"value": wl.P / (ms * 1e-3), "unit": "params/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": ms, "steps": steps, "grads": "seeded N(0, sigma) cast to the value dtype; weights finite after",
            "path": ("public API (ResidualSGD/ResidualAdamW.step, one optimizer per chunk of ~1/8 of the "
                     "parameters); pinned H2D of grads and D2H of values on copy streams, chunk by chunk, "
                     "overlapping the compute") if wl.world == 1
            else "mpo_sharded_step + pinned H2D/D2H"}


def _oracle_rate(name, threads, budget_s, n=1 << 22):
    """Params/s of the oracle as it stands on a bounded sample of the workload's recipe: n params
    (weights N(0, 0.02), the bench's gradient scale, its hyper-parameters, clip pre-pass included)
    stepped repeatedly until budget_s has passed.  threads = 1: the plain build; 0: the OpenMP build
    over every core of the affinity mask."""
    import numpy as np
    import oracle
    import synth
    wl, fmt, kind, hp, _ = WORKLOADS[name]
    used = oracle.parallel(threads != 1, 0 if threads != 1 else 1)
    try:
        w = synth.weights(n, 0.02, 0xB0B)
        h, r = oracle.split(fmt, w)
        g = synth.grads(n, 1e-3 if kind == "adam" else 1e-2, fmt, 0xB0B, 1)
        m = np.zeros(n, np.float32)
        v = np.zeros(n, np.float32)
        done, t0, steps = 0, time.perf_counter(), 0
        while True:
            steps += 1
            if kind == "sgd":
                oracle.sgd_step(fmt, fmt, h, r, g, m, lr=hp["lr"], momentum=hp["momentum"],
                                weight_decay=hp["weight_decay"], first_step=(steps == 1))
            else:
                coef = None
                if hp.get("max_grad_norm"):
                    coef = oracle.clip_coef(oracle.sumsq(fmt, g), hp["max_grad_norm"])
                oracle.adam_step(fmt, fmt, h, r, g, m, v, lr=hp["lr"], beta1=hp["beta1"], beta2=hp["beta2"],
                                 eps=hp["eps"], weight_decay=hp.get("weight_decay", 0.0), adamw=hp["adamw"],
                                 step=steps, clip_coef=coef)
            done += n
            el = time.perf_counter() - t0
            if el >= budget_s:
                break
    finally:
        oracle.parallel(False)
    return {"value": done / el, "unit": "params/s", "threads": used,
            "sample": f"{steps} steps x {n} params ({kind}, {fmt}) of the {wl} workload's recipe, {el:.1f} s"}


def cpu_baseline(name, budget_s=10.0):
    """The oracle as it stands (plain C) on this host: one thread, and the bit-identical OpenMP
    build over every core of the affinity mask (the headline `value`/`cores`)."""
    one = _oracle_rate(name, 1, budget_s)
    allc = _oracle_rate(name, 0, budget_s, n=1 << 24)
    return {"value": allc["value"], "unit": "params/s", "cores": allc["threads"], "kind": "oracle",
            "cpu": cpu_model(), "host_cores": len(os.sched_getaffinity(0)),
            "sample": allc["sample"] + f"; OpenMP build, {allc['threads']} threads",
            "threads_1": one, "threads_all": allc}


def _mem_available():
    """Bytes of MemAvailable in /proc/meminfo (None if unreadable)."""
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the CPU oracle timed on this host (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    oracle.build()
    name = args.workload
    wl, fmt, kind, hp, _ = WORKLOADS[name]
    from synth import workloads
    P = workloads.total(wl)
    # the oracle as it stands, over every host core: its OpenMP build (bit-identical to the plain one)
    threads = oracle.parallel(True, 0)
    # size each reference step so the whole --steps K --warmup W run stays within ~2 minutes
    budget = 100.0 / max(1, args.steps + args.warmup)
    probe = 1 << 20
    wp = synth.weights(probe, 0.02, 1)
    hp_, rp_ = oracle.split(fmt, wp)
    gp = synth.grads(probe, 1e-3, fmt, 1, 1)
    mp_, vp_ = np.zeros(probe, np.float32), np.zeros(probe, np.float32)
    t0 = time.perf_counter()
    oracle.adam_step(fmt, fmt, hp_, rp_, gp, mp_, vp_, lr=1e-3)
    rate = probe / (time.perf_counter() - t0)
    n = int(min(P, 1 << 27, max(8192, rate * budget)))
    n -= n % 8
    w = synth.weights(n, 0.02, 0xB0B)
    h, r = oracle.split(fmt, w)
    g = synth.grads(n, 1e-3, fmt, 0xB0B, 1)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    t = [0]

    def step():
        t[0] += 1
        if kind == "sgd":
            oracle.sgd_step(fmt, fmt, h, r, g, m, lr=hp["lr"], momentum=hp["momentum"], weight_decay=hp["weight_decay"],
                            first_step=(t[0] == 1))
        else:
            coef = oracle.clip_coef(oracle.sumsq(fmt, g), hp["max_grad_norm"]) if hp.get("max_grad_norm") else None
            oracle.adam_step(fmt, fmt, h, r, g, m, v, lr=hp["lr"], beta1=hp["beta1"], beta2=hp["beta2"], eps=hp["eps"],
                             weight_decay=hp.get("weight_decay", 0.0), adamw=hp["adamw"], step=t[0], clip_coef=coef)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    ms = el * 1e3 / args.steps
    value = n / (ms * 1e-3)
    line = {"impl": "reference", "metric": "optimizer-step params/sec", "value": value, "unit": "params/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "storage": f"{fmt} value + int16 residual, fp32 optimizer state", "data": "synthetic",
            "config": workload_config(name),
            "sample": {"params_per_step": n, "params_in_workload": P,
                       "note": "each step runs the oracle over a bounded prefix of the workload's recipe"},
            "cpu_baseline": {"value": value, "unit": "params/s", "cores": threads, "kind": "oracle", "cpu": cpu_model(),
                             "host_cores": len(os.sched_getaffinity(0)),
                             "sample": f"{n} of {P} params per step, {args.steps} steps; OpenMP build, "
                                       f"{threads} threads"},
            "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def secondary(names, steps, warmup, hbm_peak):
    import torch
    out = {}
    for name in names:
        try:
            out[name] = _secondary_one(name, steps, warmup, hbm_peak)
        except Exception as e:  # recorded, not hidden
            out[name] = {"error": f"{type(e).__name__}: {e}"}
        torch.cuda.empty_cache()
    return out


def _secondary_one(name, steps, warmup, hbm_peak, scheme="rne"):
    import torch
    if True:
        wl = Workload(name, scheme=scheme)
        use_sharded = name == "llama7b_adam"
        st = max(3, min(steps, int(2.0 / max(1e-6, wl.P * wl.bytes_per_param / (hbm_peak * 1e9)))))
        ms, launches = timed(lambda: wl.step(sharded=use_sharded), st, warmup)
        res = {"params_per_s": wl.P / (ms * 1e-3), "ms_per_step": ms, "steps": st,
                     "config": f"BASELINE configs[{wl.cfg}] parameter set {WORKLOADS[name][0]} "
                               f"({wl.P} params, {wl.ntensors} tensors), {wl.fmt} + {scheme} residual, "
                               + ("mpo_sharded_step world 1 (RS/AG degenerate)" if use_sharded else
                                  "one multi-tensor launch" + (" + norm pre-pass" if wl.clip else "")),
                     "bytes_per_param": wl.bytes_per_param,
                     "achieved_gbs_step": wl.P * wl.bytes_per_param / (ms * 1e-3) / 1e9,
                     "frac_of_measured_hbm": wl.P * wl.bytes_per_param / (ms * 1e-3) / 1e9 / hbm_peak,
                     "launches_per_step": launches / st,
                     "persistent_bytes_per_param": wl.persistent_bytes / wl.P}
        del wl
        return res


def torch_comparators_secondary(name, hbm_peak, steps=20, warmup=3):
    """SURVEY 8(a) "same-box comparators": the optimizer steps the paper's method replaces, on the
    same parameter set (one tensor per parameter shape), timed like the headline:
      * amp_fp32_master: torch's fused optimizer (Adam/AdamW/SGD, fused=True) over fp32 master
        weights with fp32 grads, then the per-iteration recast of the masters into the bf16/fp16
        model copy (the AMP inventory the paper compares with) -- Adam 28 + 6 B/param,
        SGD-momentum 20 + 6;
      * low_precision_only: the same fused optimizer directly on the 16-bit parameters with 16-bit
        grads and (torch's choice) 16-bit state: no master, lossy (the paper's "fp16" row) --
        Adam 14, SGD-momentum 10 B/param.
    Same hyper-parameters as the workload; weights N(0, 0.02), grads N(0, 1e-3), seeded."""
    import torch
    from synth import workloads
    wl, fmt, kind, hpkw, cfg = WORKLOADS[name]
    sizes = workloads.sizes(wl)
    P = sum(sizes)
    tdt = torch.float16 if fmt == "fp16" else torch.bfloat16
    if kind == "adam":
        hp = dict(lr=hpkw["lr"], betas=(hpkw["beta1"], hpkw["beta2"]), eps=hpkw["eps"],
                  weight_decay=hpkw.get("weight_decay", 0.0))
        opt_cls = torch.optim.AdamW if hpkw.get("adamw", False) else torch.optim.Adam
    else:
        hp = dict(lr=hpkw["lr"], momentum=hpkw.get("momentum", 0.0), weight_decay=hpkw.get("weight_decay", 0.0))
        opt_cls = torch.optim.SGD
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0xB0B)
    res = {"config": f"BASELINE configs[{cfg}] parameter set {wl} ({P} params, {len(sizes)} tensors), "
                     f"torch {opt_cls.__name__}(fused=True), hyper-parameters of the workload"}

    def run(master_dtype, model_dtype):
        ps = [torch.empty(n, dtype=master_dtype, device="cuda").normal_(0, 0.02, generator=gen) for n in sizes]
        for p in ps:
            p.grad = torch.empty_like(p).normal_(0, 1e-3, generator=gen)
        model = [torch.empty(n, dtype=model_dtype, device="cuda") for n in sizes] if model_dtype != master_dtype else None
        opt = opt_cls(ps, fused=True, **hp)

        def step():
            opt.step()
            if model is not None:
                torch._foreach_copy_(model, ps)      # the AMP recast of the masters into the model copy
        ms, _ = timed(step, steps, warmup)
        esz = ps[0].element_size()
        state = [t for t in opt.state[ps[0]].values() if torch.is_tensor(t) and t.numel() == ps[0].numel()]
        st = sum(t.element_size() for t in state)
        b = (2 * esz + st) + (esz + st)              # read p, g, state; write p, state
        if model is not None:
            b += esz + model[0].element_size()          # recast: read master, write model copy
        out = {"params_per_s": P / (ms * 1e-3), "ms_per_step": ms, "steps": steps, "bytes_per_param": b,
               "achieved_gbs": P * b / (ms * 1e-3) / 1e9,
               "frac_of_measured_hbm": P * b / (ms * 1e-3) / 1e9 / hbm_peak,
               "state_dtype": str(state[0].dtype).replace("torch.", "") if state else None}
        del opt, ps, model
        torch.cuda.empty_cache()
        return out

    res["amp_fp32_master"] = run(torch.float32, tdt)
    res["low_precision_only"] = run(tdt, tdt)
    return res


def split_reconstruct_secondary(hbm_peak, n=1 << 28, steps=50, warmup=5):
    """a1 / a2 (one-off conversions): mpo_split of n fp32 weights into bf16 value + int16
    residual and mpo_reconstruct back, 8 B/param each (read 4 + write 2 + 2, read 2 + 2 + write 4)."""
    import torch
    import paper_2309_12381_b200 as mpo
    w = torch.randn(n, device="cuda") * 0.02
    v = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    r = torch.empty(n, dtype=torch.int16, device="cuda")
    out = torch.empty(n, device="cuda")
    res = {}
    for name, fn in (("split", lambda: mpo.mpo_split(w, torch.bfloat16, value=v, resid=r)),
                     ("reconstruct", lambda: mpo.mpo_reconstruct(v, r, out=out))):
        ms, launches = timed(fn, steps, warmup)
        gbs = 8 * n / (ms * 1e-3) / 1e9
        res[name] = {"params_per_s": n / (ms * 1e-3), "ms": ms, "gbs": gbs, "frac_of_measured_hbm": gbs / hbm_peak,
                     "launches": launches / steps}
    # the round trip is exact except on bf16's RNE upper ties (R3: 1 binary32 ulp low, ~2^-17 of them)
    res["round_trip_inexact_fraction"] = float((out != w).float().mean().item())
    res["config"] = f"{n} fp32 weights N(0, 0.02), bf16 value + int16 residual, 8 B/param each way"
    del w, v, r, out
    torch.cuda.empty_cache()
    return res


def _single_rank_group():
    """A one-rank NCCL process group (for the sharded optimizers at world 1), once per process."""
    import socket
    import torch
    import torch.distributed as tdist
    if tdist.is_initialized():
        return
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
    sk.close()
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", torch.cuda.current_device()))


def per_tensor_secondary(name, hbm_peak, steps=50, warmup=5):
    """SURVEY 8(d) "multi-tensor vs per-tensor launch" ("too many kernel launches can hinder
    performance on smaller parameters"): the same step as one launch over the whole table, as one
    launch per tensor from Python, and as those per-tensor launches captured in a CUDA graph
    (device-side cost of the launches alone)."""
    import torch
    wl = Workload(name)
    mpo = wl.mpo
    L = wl.layout
    shapes = [(n,) for n in wl.sizes]
    V, R, G, M = (L.views(t, shapes) for t in (wl.value, wl.resid, wl.grad, wl.m))
    W = L.views(wl.v, shapes) if wl.v is not None else [None] * len(shapes)
    tabs = [mpo.TensorTable([v], [r], [g], [m], [w], scheme=wl.scheme) for v, r, g, m, w in zip(V, R, G, M, W)]

    def per_tensor():
        wl.t += 1
        hp = wl.hp()
        for t in tabs:
            (mpo.mpo_sgd_step if wl.kind == "sgd" else mpo.mpo_adam_step)(t, hp)
    ms_multi, _ = timed(wl.step, steps, warmup)
    ms_py, launches = timed(per_tensor, steps, warmup)
    g_ms = None
    try:
        s_ = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_):
            per_tensor()
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=s_):
                per_tensor()
        graph.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            graph.replay()
        b.record()
        torch.cuda.synchronize()
        g_ms = a.elapsed_time(b) / steps
        del graph
    except Exception as ex:   # recorded, not hidden
        g_ms = f"unavailable: {type(ex).__name__}: {ex}"[:200]
    per = wl.P * wl.bytes_per_param
    res = {"config": f"{name}: {wl.P} params, {wl.ntensors} tensors",
           "multi_tensor_one_launch": {"ms_per_step": ms_multi, "frac_of_measured_hbm": per / (ms_multi * 1e-3) / 1e9 / hbm_peak},
           "per_tensor_from_python": {"ms_per_step": ms_py, "launches_per_step": launches / steps,
                                      "frac_of_measured_hbm": per / (ms_py * 1e-3) / 1e9 / hbm_peak},
           "per_tensor_cuda_graph": ({"ms_per_step": g_ms, "frac_of_measured_hbm": per / (g_ms * 1e-3) / 1e9 / hbm_peak}
                                     if isinstance(g_ms, float) else g_ms)}
    del wl, tabs
    torch.cuda.empty_cache()
    return res


def flat1m_secondary(hbm_peak, steps=100, warmup=10):
    """BASELINE configs[0]: one flat 2^20-param fp16 + residual tensor, Adam, 100 steps per
    measurement.  Its 27 MB per step fits the 126 MB L2 and one launch is a few microseconds, so
    back to back it is launch/L2-bound ("too many kernel launches can hinder performance on
    smaller parameters"); rotating through >= 4 x L2 of independent parameter sets gives its
    HBM-bound number (each launch finds its set evicted)."""
    import torch
    wl = Workload("flat1m_adam")
    bpp = wl.bytes_per_param
    ms, launches = timed(wl.step, steps, warmup)
    per = wl.P * bpp
    sets = int(math.ceil(4 * L2_BYTES / per)) + 1
    pool = [wl] + [Workload("flat1m_adam", seed=0xB0B + k) for k in range(1, sets)]
    it = [0]

    def rot():
        pool[it[0] % sets].step()
        it[0] += 1
    ms_rot, _ = timed(rot, steps * 2, sets)
    # device side only: the same `steps` launches (step counts 1..steps) captured in one CUDA graph
    # and replayed, so the host's per-call cost (Python marshalling + validation + launch, ~10 us)
    # drops out and what remains is the kernel's own launch-to-launch time
    g_us = None
    try:
        s_ = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        t0_ = wl.t
        with torch.cuda.stream(s_):
            wl.step()                                   # warm (first-call attribute setup) off-graph
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=s_):
                for _ in range(steps):
                    wl.step()
        wl.t = t0_
        graph.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            graph.replay()
        b.record()
        torch.cuda.synchronize()
        g_us = a.elapsed_time(b) / (5 * steps) * 1e3
        del graph
    except Exception as ex:   # recorded, not hidden
        g_us = f"unavailable: {type(ex).__name__}: {ex}"[:200]
    # device side AND L2-flushed: the rotation over the >= 4 x L2 pool captured in one CUDA graph
    # (each launch finds its set evicted by the sets stepped since; no host cost in between)
    gr_us = None
    try:
        s_ = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        ts = [x.t for x in pool]
        it[0] = 0
        with torch.cuda.stream(s_):
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=s_):
                for _ in range(steps * 2):
                    rot()
        for x, t_ in zip(pool, ts):
            x.t = t_
        graph.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            graph.replay()
        b.record()
        torch.cuda.synchronize()
        gr_us = a.elapsed_time(b) / (5 * steps * 2) * 1e3
        del graph
    except Exception as ex:   # recorded, not hidden
        gr_us = f"unavailable: {type(ex).__name__}: {ex}"[:200]
    res = {"config": f"BASELINE configs[0]: {wl.P} params, 1 tensor, fp16 + int16 residual, Adam, {steps} steps",
           "l2_flushed_rotating_cuda_graph": ({"us_per_step": gr_us, "params_per_s": wl.P / (gr_us * 1e-6),
                                               "gbs": per / (gr_us * 1e-6) / 1e9, "frac_of_measured_hbm":
                                               per / (gr_us * 1e-6) / 1e9 / hbm_peak, "sets": sets,
                                               "note": "the HBM-bound C1 number: device only, every launch on "
                                                       "an L2-evicted set"}
                                              if isinstance(gr_us, float) else gr_us),
           "cuda_graph_device_only": ({"us_per_step": g_us, "params_per_s": wl.P / (g_us * 1e-6),
                                       "gbs": per / (g_us * 1e-6) / 1e9, "frac_of_measured_hbm":
                                       per / (g_us * 1e-6) / 1e9 / hbm_peak}
                                      if isinstance(g_us, float) else g_us),
           "bytes_per_param": bpp, "launches_per_step": launches / steps,
           "back_to_back_l2_resident": {"params_per_s": wl.P / (ms * 1e-3), "us_per_step": ms * 1e3,
                                        "gbs": per / (ms * 1e-3) / 1e9,
                                        "note": "27 MB working set < L2; bound by the host's per-call cost "
                                                "(Python marshalling + C validation + launch), see cuda_graph"},
           "l2_flushed_rotating_from_python": {"params_per_s": wl.P / (ms_rot * 1e-3), "us_per_step": ms_rot * 1e3,
                                   "gbs": per / (ms_rot * 1e-3) / 1e9,
                                   "frac_of_measured_hbm": per / (ms_rot * 1e-3) / 1e9 / hbm_peak,
                                   "sets": sets, "rotated_bytes": sets * per}}
    del pool, wl
    torch.cuda.empty_cache()
    return res


def hook_mode_secondary(steps=8, warmup=3, batch=8, seq=1024, modes=("hook", "two_phase", "amp_fp32_master")):
    """BASELINE configs[2]: GPT-2 small (HF GPT2LMHeadModel, random init, tied lm_head, 124 439 808
    params / 148 tensors) in bf16 + int16 residual, AdamW (lr 6e-4, betas (0.9, 0.95), wd 0.1)
    fused into backward through post-accumulate-grad hooks, on synthetic tokens
    (B=8, T=1024).  Compared in the same process with (a) the two-phase form: backward keeping
    16-bit grads + one multi-tensor step; (b) the paper's baseline inventory, torch AMP-style fp32
    master weights + bf16 model copy + fp32 grads + torch.optim.AdamW(fused=True).  Reports
    time per training step (fwd+bwd+update), persistent and peak bytes per parameter."""
    import torch
    import paper_2309_12381_b200 as mpo
    from transformers import GPT2Config, GPT2LMHeadModel
    dev = torch.device("cuda")
    out = {}
    gen = torch.Generator(device=dev).manual_seed(2023)
    idx = torch.randint(0, 50257, (batch, seq + 1), device=dev, generator=gen)
    # create the cuBLAS / cuBLASLt workspaces (process-wide, allocated by the first GEMM of the
    # stream through torch's allocator) before any mode's memory baseline, so that no mode is
    # charged for them
    for dt in (torch.float32, torch.bfloat16):
        a = torch.randn(256, 256, device=dev, dtype=dt, requires_grad=True)
        (a @ a).float().sum().backward()
        torch.nn.functional.linear(a, a).float().sum().backward()
        del a
    # ... and the ones the autograd engine's device thread creates for this model's shapes (its own
    # cuBLAS / cuBLASLt handle, 1 MiB Lt workspace): one throwaway fwd+bwd of the same model, so
    # that no mode is charged for them (round 1 charged 1 MiB = 0.008 B/param to the first mode)
    torch.manual_seed(0)
    warm = GPT2LMHeadModel(GPT2Config()).to(dev).to(torch.bfloat16)
    logits = warm(idx[:, :-1]).logits
    torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]), idx[:, 1:].reshape(-1)).backward()
    del warm, logits
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    def loss_of(model):
        logits = model(idx[:, :-1]).logits
        return torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]), idx[:, 1:].reshape(-1))

    def run(mode):
        import gc
        gc.collect()            # the previous mode's hooks <-> params <-> optimizer cycle
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()   # whatever an earlier mode left behind is excluded
        req = lambda: torch.cuda.memory_stats().get("requested_bytes.all.current", 0)
        base_req = req()
        torch.manual_seed(0)
        model = GPT2LMHeadModel(GPT2Config()).to(dev)
        P = sum(p.numel() for p in model.parameters())
        hp = dict(lr=6e-4, betas=(0.9, 0.95), weight_decay=0.1)
        if mode in ("hook", "hook_python", "two_phase"):
            opt = mpo.ResidualAdamW(model.parameters(), fmt=torch.bfloat16, **hp)   # splits fp32 init on the GPU
            if mode == "hook":
                opt.install_backward_hooks()                 # native (C++) hooks
            elif mode == "hook_python":
                opt.install_backward_hooks(native=False)     # the same logic as Python hooks (A/B)

            def step(rec=None):
                loss = loss_of(model)
                if rec is not None:
                    rec[0].record()
                loss.backward()
                if rec is not None:
                    rec[1].record()
                if mode == "two_phase":
                    opt.step()
                    for p in model.parameters():
                        p.grad = None
                return loss
        elif mode == "two_phase_graph":
            # the whole training iteration -- forward, backward, the residual AdamW step -- captured
            # once as a CUDA graph and replayed (the step's hyper-parameters travel through the
            # pinned block of mpo_step_graphed): no per-kernel host cost at all
            opt = mpo.ResidualAdamW(model.parameters(), fmt=torch.bfloat16, **hp)
            x_in, y_in = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()

            def loss_static():
                logits = model(x_in).logits
                return torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]),
                                                         y_in.reshape(-1))
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):       # warm-up: every gradient buffer allocated once
                for _ in range(2):
                    loss_static().backward()
            torch.cuda.current_stream().wait_stream(side)
            opt.enable_graph_step()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for p in model.parameters():
                    p.grad.zero_()
                loss_g = loss_static()
                loss_g.backward()
                opt.step()

            def step(rec=None):
                opt.prepare_step()
                if rec is not None:
                    rec[0].record()
                graph.replay()
                if rec is not None:
                    rec[1].record()
                return loss_g
        elif mode in ("sharded_two_phase", "sharded_bucketed"):
            # hook mode x sharding at world 1: bucket steps issued from the hooks
            # on a side stream overlap the rest of backward, vs backward + one sharded step
            _single_rank_group()
            mk = mpo.BucketedShardedOptimizer if mode == "sharded_bucketed" else mpo.ShardedResidualOptimizer
            b1, b2 = hp["betas"]
            ahp = mpo.AdamParams(lr=hp["lr"], beta1=b1, beta2=b2, weight_decay=hp["weight_decay"])
            kw = {"bucket_elems": 1 << 24} if mode == "sharded_bucketed" else {}
            opt = mk(list(model.parameters()), kind="adam", fmt=torch.bfloat16, hp=ahp, **kw)

            def step(rec=None):
                loss = loss_of(model)
                if rec is not None:
                    rec[0].record()
                loss.backward()
                if mode == "sharded_bucketed":
                    opt.wait()
                if rec is not None:
                    rec[1].record()
                if mode == "sharded_two_phase":
                    opt.step()
                    opt.zero_grad()
                return loss
        else:   # paper's baseline: fp32 master + bf16 working copy + fp32 grads + fused AdamW
            master = [p.detach().clone().float() for p in model.parameters()]
            model = model.to(torch.bfloat16)
            opt = torch.optim.AdamW(master, fused=True, **hp)
            params = list(model.parameters())

            def step(rec=None):
                loss = loss_of(model)
                if rec is not None:
                    rec[0].record()
                loss.backward()
                if rec is not None:
                    rec[1].record()
                for m_, p in zip(master, params):
                    m_.grad = p.grad.float()
                    p.grad = None
                opt.step()
                opt.zero_grad(set_to_none=False)
                with torch.no_grad():
                    for m_, p in zip(master, params):
                        p.copy_(m_)
                return loss
        torch.cuda.synchronize()
        state = torch.cuda.memory_allocated() - base   # params + residual/master + optimizer state
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        persistent = torch.cuda.memory_allocated() - base   # what survives between training steps
        # the same without the caching allocator's block rounding (requested sizes)
        persistent_req = req() - base_req
        torch.cuda.reset_peak_memory_stats()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            loss = step()
        e.record()
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base
        # phase breakdown (separate steps, so the events do not perturb the number above):
        # forward, backward (hook mode: with its fused steps), the rest (two-phase: the step)
        ph = [0.0, 0.0, 0.0]
        for _ in range(steps):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            step(rec=ev[1:3])
            ev[3].record()
            torch.cuda.synchronize()
            for k in range(3):
                ph[k] += ev[k].elapsed_time(ev[k + 1]) / steps
        hook_kernels_ms = None
        if mode == "hook":
            # summed device time of this library's kernels inside one hook-mode training step
            # (CUPTI through torch.profiler; nsys is not installed in this image)
            try:
                from torch.profiler import ProfilerActivity, profile
                with profile(activities=[ProfilerActivity.CUDA]) as prof:
                    step()
                    torch.cuda.synchronize()
                hook_kernels_ms = sum(e.self_device_time_total for e in prof.key_averages()
                                      if "mpo::" in e.key) / 1e3
            except Exception as ex:   # recorded, not hidden
                hook_kernels_ms = f"unavailable: {type(ex).__name__}: {ex}"[:200]
        res = {"ms_per_train_step": s.elapsed_time(e) / steps, "forward_ms": ph[0], "backward_ms": ph[1],
               "after_backward_ms": ph[2], "library_kernels_ms_per_step": hook_kernels_ms,
               "state_bytes_per_param": state / P,
               "persistent_bytes_per_param": persistent / P,
               "persistent_requested_bytes_per_param": persistent_req / P,
               "peak_bytes_per_param": peak / P, "peak_gb": peak / 1e9, "loss": float(loss.detach()), "leftover_bytes_excluded": base}
        del model, opt, step, loss
        return res
    for mode in modes:
        try:
            out[mode] = run(mode)
        except Exception as ex:   # recorded, not hidden
            out[mode] = {"error": f"{type(ex).__name__}: {ex}"}
    try:
        out["persistent_saving_vs_amp_bytes_per_param"] = {
            "allocated": out["amp_fp32_master"]["persistent_bytes_per_param"] - out["hook"]["persistent_bytes_per_param"],
            "requested": (out["amp_fp32_master"]["persistent_requested_bytes_per_param"]
                          - out["hook"]["persistent_requested_bytes_per_param"])}
    except Exception:
        pass
    try:   # SURVEY 8(d)'s three hook-mode numbers (+3-4 % time in the paper)
        h, t = out["hook"], out["two_phase"]
        out["hook_breakdown"] = {
            "added_backward_ms": h["backward_ms"] - t["backward_ms"],
            "hook_kernels_ms": h["library_kernels_ms_per_step"],
            "two_phase_backward_plus_step_ms": t["backward_ms"] + t["after_backward_ms"],
            "hook_backward_ms": h["backward_ms"],
            "hook_vs_two_phase_train_step": h["ms_per_train_step"] / t["ms_per_train_step"] - 1.0}
    except Exception:
        pass
    try:   # the same iteration as one CUDA graph (mpo_step_graphed) vs eager
        out["graph_vs_eager_two_phase"] = out["two_phase_graph"]["ms_per_train_step"] / out["two_phase"]["ms_per_train_step"]
    except Exception:
        pass
    try:   # hook mode x sharding at world 1: bucket steps overlapping backward vs a step after it
        b_, t_ = out["sharded_bucketed"], out["sharded_two_phase"]
        out["bucketed_sharding_world1"] = {
            "bucketed_train_step_ms": b_["ms_per_train_step"], "two_phase_sharded_train_step_ms": t_["ms_per_train_step"],
            "two_phase_step_after_backward_ms": t_["after_backward_ms"],
            "bucketed_vs_two_phase": b_["ms_per_train_step"] / t_["ms_per_train_step"] - 1.0}
    except Exception:
        pass
    out["config"] = (f"BASELINE configs[2]: HF GPT2LMHeadModel random init (124439808 params, 148 tensors), "
                     f"synthetic tokens B={batch} T={seq}, AdamW lr 6e-4 betas (0.9,0.95) wd 0.1; time = fwd+bwd+update")
    return out


_JSON_OUT = None


def _claim_stdout():
    """Keep stdout for the one JSON line: libraries that print to fd 1 (NCCL's version banner on
    communicator creation, for one) are redirected to stderr for the rest of the run."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
        sys.stdout = sys.stderr


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)      # ~1.2 s timed region at the LLaMA-7B step
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mpo", choices=["mpo", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--no-p2p", action="store_true",
                    help="N>1 (or --mg-breakdown): skip the P2P / NVLS fused sharded steps on torch symmetric memory")
    ap.add_argument("--mg-breakdown", action="store_true",
                    help="run the N>1 update/collective breakdown at world 1 too (code-path check)")
    ap.add_argument("--fused-child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if args.fused_child:
        return fused_child(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2309_12381_b200 import _build
    _build.build()
    hbm_peak, peak_src = peaks()

    wl = Workload(args.workload, world, rank)
    sampler = ClockSampler(local) if rank == 0 else None
    ms, launches = timed(wl.step, args.steps, args.warmup, dist, sampler)
    # one step-kernel launch per step at N=1 without clipping: the region time per launch IS the
    # kernel's mean launch duration; with clipping the step also holds the norm pre-pass (2 small
    # launches), and at N>1 the NCCL collectives, so the whole step is reported (its bytes include
    # the grad re-read: 28 B/param)
    per_launch = ms
    clocks = sampler.stop() if sampler else None
    value = wl.P / (ms * 1e-3)
    n_upd = wl.layout.shard if world > 1 else wl.P
    alg_bytes = n_upd * wl.bytes_per_param
    # dominant kernel: at N=1 the step is one launch of the step kernel; at N>1 the step window
    # also holds the NCCL collectives, so the kernel's own time comes from the update-only
    # measurement of multi_gpu_breakdown below.
    achieved = alg_bytes / (per_launch * 1e-3) / 1e9
    traffic = ncu_traffic(args.workload) if world == 1 else None   # the committed capture is of the N=1 launch
    box_copy = None
    try:
        if world == 1 and torch.cuda.mem_get_info()[0] > 5 * (1 << 30):   # two 2 GiB buffers
            box_copy = same_box_copy_gbs()
    except Exception:
        box_copy = None
    mg = None
    if world > 1 or args.mg_breakdown:
        try:
            if dist is None:   # --mg-breakdown at world 1: the single-rank NCCL group (code-path check)
                import torch.distributed as tdist
                wl.step(sharded=True)
                dist = tdist
            mg = multi_gpu_breakdown(wl, dist, args.steps, args.warmup, p2p=not args.no_p2p)
            if world > 1:
                # the step kernel's own launch time on the shard (the whole-step window also
                # holds the NCCL collectives, reported with their NVLink fractions in multi_gpu)
                per_launch = mg["update_only"]["ms_per_step"]
                achieved = alg_bytes / (per_launch * 1e-3) / 1e9
        except Exception as ex:   # reported, never fatal to the JSON line
            mg = {"error": f"{type(ex).__name__}: {ex}"}
    # at N=1 the e2e leg builds its own parameters / optimizer: release this workload's device
    # buffers first (the LLaMA-7B set would not fit twice); at N>1 it steps this workload
    if world == 1:
        wl.release()
    e2e = e2e_measure(wl, min(args.e2e_steps, args.steps), dist)
    line = {
        "metric": "optimizer-step params/sec", "value": value, "unit": "params/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f32", "storage": f"{wl.fmt} value + int16 residual, fp32 optimizer state", "data": "synthetic",
        "config": workload_config(args.workload),
        "path": "mpo_sharded_step (NCCL RS -> shard update -> NCCL AG)" if world > 1
                else "mpo_sgd_step/mpo_adam_step, one multi-tensor launch",
        "parallelism": f"dp{world} sharded optimizer state" if world > 1 else "single GPU",
        "l2": f"working set {alg_bytes / 1e6:.0f} MB/step > L2 {L2_BYTES / 2**20:.0f} MiB (no flush)",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                     "frac_of_8tbs_spec": achieved / 8000.0,
                     "kernel": "step_tma_kernel (reconstruct -> update -> re-split)",
                     "algorithmic_bytes_per_launch": alg_bytes, "bytes_per_param": wl.bytes_per_param,
                     "mean_launch_ms": per_launch, "same_box_copy_gbs": box_copy,
                     "frac_of_same_box_copy": (achieved / box_copy) if box_copy else None},
        "gpu_launches": launches,
        **({"multi_gpu": mg} if mg is not None else {}),
        "clocks": clocks,
        "e2e": e2e,
        "memory": {"persistent_bytes_per_param": wl.persistent_bytes / wl.P,
                   "paper_amp_inventory_bytes_per_param": 14 if wl.kind == "sgd" else 18,
                   "note": "multi-tensor mode keeps a 16-bit grad buffer (2 B); hook mode keeps none"},
    }
    if rank == 0 and world == 1 and not args.no_secondary:
        del wl
        torch.cuda.empty_cache()
        line["secondary"] = secondary([n for n in ("resnet50_sgd", "resnet50_sgd_plain", "gpt2_adamw",
                                                   "vit_l16_adam_clip", "llama7b_adam")
                                       if n != args.workload], 200, 5, hbm_peak)
        if args.workload == "llama7b_adam":
            # the same LLaMA-7B step through the sharded entry point at world 1 (one flat piece, the
            # NCCL reduce-scatter / all-gather issued as single-rank no-ops): the N>1 path's cost at N=1
            try:
                line["secondary"]["llama7b_adam_sharded_world1"] = _secondary_one("llama7b_adam", 20, 3, hbm_peak)
            except Exception as ex:
                line["secondary"]["llama7b_adam_sharded_world1"] = {"error": f"{type(ex).__name__}: {ex}"}
            torch.cuda.empty_cache()
        try:
            line["secondary"]["resnet50_multi_vs_per_tensor"] = per_tensor_secondary("resnet50_sgd", hbm_peak)
        except Exception as ex:
            line["secondary"]["resnet50_multi_vs_per_tensor"] = {"error": f"{type(ex).__name__}: {ex}"}
        for cname, mpo_ms in (("resnet50_sgd", line["secondary"].get("resnet50_sgd", {}).get("ms_per_step")),
                              ("gpt2_adamw", line["secondary"].get("gpt2_adamw", {}).get("ms_per_step")),
                              ("llama7b_adam", ms if args.workload == "llama7b_adam" else None)):
            try:
                cmp_ = torch_comparators_secondary(cname, hbm_peak)
                if isinstance(mpo_ms, float):
                    cmp_["mpo_step_ms"] = mpo_ms
                    cmp_["mpo_speedup_vs_amp_fp32_master"] = cmp_["amp_fp32_master"]["ms_per_step"] / mpo_ms
                    cmp_["mpo_speedup_vs_low_precision_only"] = cmp_["low_precision_only"]["ms_per_step"] / mpo_ms
                line["secondary"][f"torch_fused_{cname}"] = cmp_
            except Exception as ex:
                line["secondary"][f"torch_fused_{cname}"] = {"error": f"{type(ex).__name__}: {ex}"}
            torch.cuda.empty_cache()
        try:
            line["secondary"]["flat1m_adam"] = flat1m_secondary(hbm_peak)
        except Exception as ex:
            line["secondary"]["flat1m_adam"] = {"error": f"{type(ex).__name__}: {ex}"}
        try:
            line["secondary"]["split_reconstruct"] = split_reconstruct_secondary(hbm_peak)
        except Exception as ex:
            line["secondary"]["split_reconstruct"] = {"error": f"{type(ex).__name__}: {ex}"}
        for sch in ("rtz", "sr", "x8", "x8z"):    # paper variants of the storage scheme, GPT-2 AdamW set
            name = "gpt2_adamw"
            fmt_ok = sch != "sr" or WORKLOADS[name][1] == "fp16"
            key = f"{name}_{sch}" + ("" if fmt_ok else "_fp16")
            try:
                if not fmt_ok:   # SR is defined for fp16: same parameter set in fp16
                    WORKLOADS["gpt2_adamw_fp16"] = ("gpt2_small", "fp16") + WORKLOADS[name][2:]
                    name = "gpt2_adamw_fp16"
                line["secondary"][key] = _secondary_one(name, 200, 5, hbm_peak, scheme=sch)
            except Exception as ex:
                line["secondary"][key] = {"error": f"{type(ex).__name__}: {ex}"}
            torch.cuda.empty_cache()
        try:
            line["secondary"]["gpt2_hook_mode"] = hook_mode_secondary(
                modes=("hook", "two_phase", "amp_fp32_master", "sharded_two_phase", "sharded_bucketed"))
        except Exception as ex:
            line["secondary"]["gpt2_hook_mode"] = {"error": f"{type(ex).__name__}: {ex}"}
        try:   # small activations (B=1, T=128): gradients are a large share of the peak
            line["secondary"]["gpt2_hook_mode_b1_t128"] = hook_mode_secondary(
                steps=20, batch=1, seq=128,
                modes=("hook", "two_phase", "amp_fp32_master", "hook_python", "two_phase_graph"))
        except Exception as ex:
            line["secondary"]["gpt2_hook_mode_b1_t128"] = {"error": f"{type(ex).__name__}: {ex}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        emit(line)
    import torch.distributed as tdist
    if tdist.is_initialized():   # the N>1 group, or the single-rank group of the world-1 sharded secondaries
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
