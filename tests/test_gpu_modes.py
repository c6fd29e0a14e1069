"""GPU: the three delivery modes agree bitwise (SURVEY 8(c) pin P8) and the optimizer objects
behave as documented.

* hook mode (step inside backward from post-accumulate-grad hooks) == two-phase
  backward + multi-tensor step, with no gradient left allocated after backward;
* sharded step (RS -> shard update -> AG over NCCL) at world_size 1 == unsharded step;
* the user-facing optimizers reproduce the oracle (exact build).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.nn as nn

import synth
from gpu_util import host16, same_bits_nan_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_12381_b200 as m
    from paper_2309_12381_b200 import _build
    _build.build()
    return m


class TinyLM(nn.Module):
    """GPT-like toy with a tied embedding / output matrix (weight sharing)."""

    def __init__(self, vocab=257, d=64):
        super().__init__()
        self.emb = nn.Embedding(vocab, d)
        self.ln = nn.LayerNorm(d)
        self.fc1 = nn.Linear(d, 4 * d)
        self.fc2 = nn.Linear(4 * d, d)

    def forward(self, idx):
        x = self.emb(idx)
        x = x + self.fc2(torch.nn.functional.gelu(self.fc1(self.ln(x))))
        return x @ self.emb.weight.t()


def _loss(model, idx):
    logits = model(idx[:, :-1]).float()
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), idx[:, 1:].reshape(-1))


def _pair(fmt, kind, mpo, **kw):
    torch.manual_seed(0)
    a = TinyLM().cuda()
    b = TinyLM().cuda()
    b.load_state_dict(a.state_dict())
    mk = (lambda ps: mpo.ResidualAdamW(ps, fmt=fmt, **kw)) if kind == "adam" else \
        (lambda ps: mpo.ResidualSGD(ps, fmt=fmt, **kw))
    return a, b, mk(a.parameters()), mk(b.parameters())


@pytest.mark.parametrize("fmt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("kind", ["adam", "sgd"])
@pytest.mark.parametrize("batch_below", [0, 1 << 16, 1 << 30])
@pytest.mark.parametrize("native", [True, False])
def test_hook_mode_equals_two_phase(mpo, fmt, kind, batch_below, native):
    """Per-parameter launches (batch_below=0), small parameters batched into one launch at the end
    of backward (default), and everything batched: all bitwise equal to the two-phase step, with
    the native (C++) hooks and with the Python hooks."""
    kw = dict(lr=1e-3, weight_decay=0.1) if kind == "adam" else dict(lr=0.1, momentum=0.9, weight_decay=1e-4)
    a, b, oa, ob = _pair(fmt, kind, mpo, **kw)
    ob.install_backward_hooks(batch_below=batch_below, native=native)
    gen = torch.Generator(device="cuda").manual_seed(1)
    for step in range(4):
        idx = torch.randint(0, 257, (4, 33), device="cuda", generator=gen)
        la = _loss(a, idx)
        la.backward()
        oa.step()
        for p in a.parameters():
            p.grad = None
        lb = _loss(b, idx)
        assert torch.equal(la, lb)          # same weights going in
        lb.backward()
        for p in b.parameters():
            assert p.grad is None           # consumed and freed inside backward
    for (na, pa), (nb, pb) in zip(a.named_parameters(), b.named_parameters()):
        assert torch.equal(pa.view(torch.int16), pb.view(torch.int16)), na
        sa, sb = oa.state[pa], ob.state[pb]
        assert torch.equal(sa["resid"], sb["resid"]), na
        assert sa["step"] == sb["step"] == 4
        for k in ("m", "v"):
            if sa.get(k) is not None:
                assert torch.equal(sa[k], sb[k]), (na, k)


def test_native_hooks_follow_lr_changes_and_uninstall(mpo):
    """An LR schedule that writes param_groups[i]["lr"] between backwards reaches the native hooks
    (their group structs are pushed on assignment); the steps equal the two-phase optimizer's;
    remove_backward_hooks() leaves ordinary gradient accumulation and keeps the step counts."""
    a, b, oa, ob = _pair(torch.bfloat16, "adam", mpo, lr=1e-3, weight_decay=0.1)
    ob.install_backward_hooks()
    sa = torch.optim.lr_scheduler.StepLR(oa, step_size=1, gamma=0.5)
    sb = torch.optim.lr_scheduler.StepLR(ob, step_size=1, gamma=0.5)
    gen = torch.Generator(device="cuda").manual_seed(2)
    for step in range(3):
        idx = torch.randint(0, 257, (4, 33), device="cuda", generator=gen)
        _loss(a, idx).backward()
        oa.step()
        for p in a.parameters():
            p.grad = None
        _loss(b, idx).backward()
        sa.step(); sb.step()
    assert ob.native_hook_calls() > 0
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert torch.equal(pa.view(torch.int16), pb.view(torch.int16))
    ob.remove_backward_hooks()
    assert all(st["step"] == 3 for st in ob.state_dict()["state"].values())
    _loss(b, idx).backward()
    assert all(p.grad is not None for p in b.parameters())


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_native_hooks_param_groups(mpo, kind):
    """Two param groups with different hyper-parameters (no decay on 1-D tensors, a different lr):
    the native hooks pick each parameter's group struct; == two-phase bitwise; installing twice is
    refused."""
    torch.manual_seed(3)
    a, b = TinyLM().cuda(), TinyLM().cuda()
    b.load_state_dict(a.state_dict())

    def groups(m):
        dec = [p for p in m.parameters() if p.dim() > 1]
        nod = [p for p in m.parameters() if p.dim() <= 1]
        if kind == "adam":
            return [{"params": dec, "weight_decay": 0.1}, {"params": nod, "weight_decay": 0.0, "lr": 3e-3}]
        return [{"params": dec, "weight_decay": 1e-4}, {"params": nod, "weight_decay": 0.0, "lr": 0.2}]
    mk = (lambda m: mpo.ResidualAdamW(groups(m), lr=1e-3, fmt=torch.bfloat16)) if kind == "adam" else \
        (lambda m: mpo.ResidualSGD(groups(m), lr=0.1, momentum=0.9, fmt=torch.bfloat16))
    oa, ob = mk(a), mk(b)
    ob.install_backward_hooks()
    with pytest.raises(mpo.MpoError):
        ob.install_backward_hooks()
    gen = torch.Generator(device="cuda").manual_seed(4)
    for _ in range(3):
        idx = torch.randint(0, 257, (4, 33), device="cuda", generator=gen)
        _loss(a, idx).backward()
        oa.step()
        for p in a.parameters():
            p.grad = None
        _loss(b, idx).backward()
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert torch.equal(pa.view(torch.int16), pb.view(torch.int16))


def test_hook_mode_refuses_clipping(mpo):
    a = TinyLM().cuda()
    opt = mpo.ResidualAdamW(a.parameters(), fmt=torch.bfloat16, max_grad_norm=1.0)
    with pytest.raises(mpo.MpoError, match="P:186"):
        opt.install_backward_hooks()


def test_hook_mode_peak_gradient_memory(mpo):
    """No gradient buffer persists: after backward nothing is held, and backward's peak is below
    the two-phase peak by roughly the gradient bytes."""
    torch.manual_seed(0)
    d = 1024
    make = lambda: nn.Sequential(*[nn.Linear(d, d, bias=False) for _ in range(8)]).cuda()
    a, b = make(), make()
    b.load_state_dict(a.state_dict())
    oa = mpo.ResidualAdamW(a.parameters(), fmt=torch.bfloat16)
    ob = mpo.ResidualAdamW(b.parameters(), fmt=torch.bfloat16)
    ob.install_backward_hooks()
    x = torch.randn(64, d, device="cuda", dtype=torch.bfloat16)
    peaks = []
    for model, opt, hooks in ((a, oa, False), (b, ob, True)):
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        model(x).float().square().mean().backward()
        if not hooks:
            opt.step()
        torch.cuda.synchronize()
        peaks.append(torch.cuda.max_memory_allocated() - base)
        held = sum(p.grad.numel() * 2 for p in model.parameters() if p.grad is not None)
        assert held == (0 if hooks else 8 * d * d * 2)
    grad_bytes = 8 * d * d * 2
    assert peaks[0] - peaks[1] >= grad_bytes - 2 * d * d * 2


def test_optimizer_matches_oracle(mpo, orc):
    """ResidualAdamW / ResidualSGD on fp32 init (split on the GPU) == oracle, 3 steps, exact build."""
    fmt = "bf16"
    n = 10007
    w = synth.weights(n, 0.02, 0xB0B)
    for kind in ("adam", "sgd"):
        p = nn.Parameter(torch.from_numpy(w.copy()).cuda())
        if kind == "adam":
            opt = mpo.ResidualAdamW([p], lr=1e-3, betas=(0.9, 0.95), weight_decay=0.1, fmt=torch.bfloat16,
                                    exact=True)
        else:
            opt = mpo.ResidualSGD([p], lr=0.05, momentum=0.9, nesterov=True, fmt=torch.bfloat16, exact=True)
        h, r = orc.split(fmt, w)
        m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
        for t in range(1, 4):
            g = synth.grads(n, 1e-2, fmt, 0xB0B, t)
            p.grad = torch.from_numpy(g.view(np.int16).copy()).view(torch.bfloat16).cuda()
            opt.step()
            if kind == "adam":
                orc.adam_step(fmt, fmt, h, r, g, m, v, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1,
                              adamw=True, step=t)
            else:
                orc.sgd_step(fmt, fmt, h, r, g, m, lr=0.05, momentum=0.9, nesterov=True, first_step=(t == 1))
        assert np.array_equal(host16(p.data), h)
        assert np.array_equal(opt.state[p]["resid"].cpu().numpy(), r)
        w32 = opt.fp32_params()[0].cpu().numpy()
        assert np.array_equal(w32.view(np.uint32), orc.reconstruct(fmt, h, r).view(np.uint32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl1():
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["adam", "sgd"])
@pytest.mark.parametrize("clip", [False, True])
def test_sharded_world1_equals_unsharded(mpo, nccl1, kind, clip):
    if kind == "sgd" and clip:
        pytest.skip("clipping is an Adam option")
    torch.manual_seed(3)
    shapes = [(33, 17), (4096,), (5,), (128, 64)]
    src = [torch.randn(s, device="cuda") * 0.02 for s in shapes]
    pa = [nn.Parameter(t.clone()) for t in src]
    pb = [nn.Parameter(t.clone()) for t in src]
    if kind == "adam":
        ref = mpo.ResidualAdamW(pa, lr=1e-3, weight_decay=0.1, fmt=torch.bfloat16,
                                max_grad_norm=0.05 if clip else None)
    else:
        ref = mpo.ResidualSGD(pa, lr=0.1, momentum=0.9, fmt=torch.bfloat16)
    if kind == "adam":   # SURVEY 8(b)'s torch-style names over the same optimizer
        sh = mpo.ShardedResidualAdamW(pb, lr=1e-3, weight_decay=0.1, fmt=torch.bfloat16,
                                      max_grad_norm=0.05 if clip else None)
    else:
        sh = mpo.ShardedResidualSGD(pb, lr=0.1, momentum=0.9, fmt=torch.bfloat16)
    for t in range(3):
        grads = [torch.randn(s, device="cuda").to(torch.bfloat16) * 1e-2 for s in shapes]
        if clip:   # exact-sum construction: every |g| = 2^-7, so S is exact in any order (P8)
            grads = [torch.sign(g) * 2.0 ** -7 + (g == 0) * 2.0 ** -7 for g in grads]
            grads = [g.to(torch.bfloat16) for g in grads]
        for p, g in zip(pa, grads):
            p.grad = g.clone()
        sh.zero_grad()
        for p, g in zip(pb, grads):
            p.grad.copy_(g)
        ref.step()
        sh.step()
    for a, b in zip(pa, pb):
        assert torch.equal(a.data.view(torch.int16), b.data.view(torch.int16))


@pytest.mark.parametrize("clip", [False, True])
@pytest.mark.parametrize("scheme", ["rne", "x8z"])
def test_sharded_grouped_world1_equals_param_groups(mpo, nccl1, clip, scheme):
    """Per-parameter hyper-parameter groups in the sharded step (mpo_sharded_step_grouped: the
    shard's pieces as a segment table; P:19 unchanged hyper-parameters, e.g. no decay on 1-D
    tensors) == ResidualAdamW with the same two param groups, bitwise at world 1; the
    communicator reports healthy (mpo_comm_check)."""
    torch.manual_seed(4)
    shapes = [(33, 17), (4096,), (5,), (128, 64), (1000,)]
    src = [torch.randn(s, device="cuda") * 0.02 for s in shapes]
    pa = [nn.Parameter(t.clone()) for t in src]
    pb = [nn.Parameter(t.clone()) for t in src]
    decay = [len(s) == 2 for s in shapes]
    mg = 0.05 if clip else None
    ref = mpo.ResidualAdamW([{"params": [p for p, d in zip(pa, decay) if d], "weight_decay": 0.1},
                             {"params": [p for p, d in zip(pa, decay) if not d], "weight_decay": 0.0}],
                            lr=1e-3, fmt=torch.bfloat16, max_grad_norm=mg, scheme=scheme)
    hps = [mpo.AdamParams(lr=1e-3, weight_decay=0.1, max_grad_norm=mg or 0.0),
           mpo.AdamParams(lr=1e-3, weight_decay=0.0, max_grad_norm=mg or 0.0)]
    sh = mpo.ShardedResidualOptimizer(pb, kind="adam", fmt=torch.bfloat16, hp=hps,
                                      hp_index=[0 if d else 1 for d in decay], scheme=scheme)
    assert len(sh.segments) > 1
    for t in range(3):
        grads = [torch.randn(s, device="cuda").to(torch.bfloat16) * 1e-2 for s in shapes]
        if clip:   # exact-sum construction (P8)
            grads = [(torch.sign(g) * 2.0 ** -7 + (g == 0) * 2.0 ** -7).to(torch.bfloat16) for g in grads]
        for p, g in zip(pa, grads):
            p.grad = g.clone()
        sh.zero_grad()
        for p, g in zip(pb, grads):
            p.grad.copy_(g)
        ref.step()
        sh.step()
        sh.check_comm()
    for a, b in zip(pa, pb):
        assert torch.equal(a.data.view(torch.int16), b.data.view(torch.int16))


@pytest.mark.parametrize("kind", ["adam", "sgd"])
@pytest.mark.parametrize("bucketed", [False, True])
@pytest.mark.parametrize("scheme", ["sr", "x8z"])
def test_sharded_resume_is_bit_identical(mpo, nccl1, kind, bucketed, scheme):
    """Checkpoint / resume of the sharded optimizers (R17): 3 steps -> torch.save(values, optimizer
    shard state) -> fresh parameters + optimizer -> load -> 3 steps == 6 uninterrupted, bitwise."""
    import io
    shapes = [(33, 17), (4096,), (5,), (128, 64)]
    torch.manual_seed(21)
    src = [torch.randn(s, device="cuda") * 0.02 for s in shapes]
    grads = [[(torch.randn(s, device="cuda") * 1e-2).to(torch.float16) for s in shapes] for _ in range(6)]
    hp = (lambda: mpo.AdamParams(lr=1e-3, weight_decay=0.1)) if kind == "adam" else \
        (lambda: mpo.SgdParams(lr=0.05, momentum=0.9))

    def make(init):
        ps = [nn.Parameter(t.clone()) for t in init]
        if bucketed:
            return ps, mpo.BucketedShardedOptimizer(ps, kind=kind, fmt=torch.float16, hp=hp(), bucket_elems=2048,
                                                    scheme=scheme, seed=3)
        return ps, mpo.ShardedResidualOptimizer(ps, kind=kind, fmt=torch.float16, hp=hp(), scheme=scheme, seed=3)

    def run(ps, opt, steps):
        for g in steps:
            if bucketed:
                # the hooks step each bucket as its last gradient is accumulated
                sum(((p.float() * gg.float()).sum() for p, gg in zip(ps, g))).backward()
                opt.wait()
            else:
                opt.zero_grad()
                for p, gg in zip(ps, g):
                    p.grad.copy_(gg)
                opt.step()
        torch.cuda.synchronize()

    pa, oa = make(src)
    run(pa, oa, grads)
    pb, ob = make(src)
    run(pb, ob, grads[:3])
    buf = io.BytesIO()
    torch.save({"value": ob.value.clone(), "opt": ob.state_dict()}, buf)
    if bucketed:
        ob.remove_hooks()
    del pb, ob
    buf.seek(0)
    ck = torch.load(buf, weights_only=False)
    pc, oc = make([torch.randn_like(t) for t in src])          # different init: all state from the file
    with torch.no_grad():
        oc.value.copy_(ck["value"])
    oc.load_state_dict(ck["opt"])
    run(pc, oc, grads[3:])
    assert oc.step_count == oa.step_count == 6
    assert torch.equal(oa.value.view(torch.int16), oc.value.view(torch.int16))
    assert torch.equal(oa.resid, oc.resid)
    for x, y in ((oa.m, oc.m), (oa.v, oc.v)):
        if x is not None:
            assert torch.equal(x, y)
    if bucketed:
        oa.remove_hooks(); oc.remove_hooks()


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_sharded_p2p_transport_world1_equals_nccl(mpo, nccl1, kind):
    """transport='p2p' (torch symmetric memory + mpo_p2p_sharded_step between symmetric-memory
    barriers) == transport='nccl' bitwise at world 1 in the exact build (the fp32 sum of one
    rank's gradient is its exact widening, R15)."""
    try:
        import torch.distributed._symmetric_memory as symm
        t = symm.empty(16, dtype=torch.bfloat16, device="cuda")
        from paper_2309_12381_b200.sharded import _rendezvous
        _rendezvous(t, None)
    except Exception as e:   # pragma: no cover - depends on the box
        pytest.skip(f"torch symmetric memory unavailable here: {type(e).__name__}: {e}")
    torch.manual_seed(5)
    shapes = [(33, 17), (4096,), (5,), (128, 64)]
    src = [torch.randn(s, device="cuda") * 0.02 for s in shapes]
    pa = [nn.Parameter(t.clone()) for t in src]
    pb = [nn.Parameter(t.clone()) for t in src]
    if kind == "adam":
        mk = lambda: mpo.AdamParams(lr=1e-3, weight_decay=0.1)
    else:
        mk = lambda: mpo.SgdParams(lr=0.1, momentum=0.9)
    # exact builds: the two kernels are different instantiations (16-bit vs fp32 gradient ingest),
    # which the FMA build may contract differently (R12)
    a = mpo.ShardedResidualOptimizer(pa, kind=kind, fmt=torch.bfloat16, hp=mk(), exact=True)
    b = mpo.ShardedResidualOptimizer(pb, kind=kind, fmt=torch.bfloat16, hp=mk(), transport="p2p", exact=True)
    for t in range(3):
        grads = [torch.randn(s, device="cuda").to(torch.bfloat16) * 1e-2 for s in shapes]
        for opt, ps in ((a, pa), (b, pb)):
            opt.zero_grad()
            for p, g in zip(ps, grads):
                p.grad.copy_(g)
            opt.step()
    torch.cuda.synchronize()
    for x, y in zip(pa, pb):
        assert torch.equal(x.data.view(torch.int16), y.data.view(torch.int16))
    assert torch.equal(a.resid, b.resid)


# ---------------------------------------------------------------------------------------------
# Gradient surgery through the optimizer: clip-by-value, loss-scale found-inf
# ---------------------------------------------------------------------------------------------
def test_clip_value_multi_tensor_and_hook_match_oracle(mpo, orc):
    """clip_value fused into the step: multi-tensor (exact build) == oracle bitwise; hook mode ==
    multi-tensor bitwise."""
    from gpu_util import dev16
    fmt = "bf16"
    sizes = [4096 + 40, 333, 8192]
    for kind in ("adam", "sgd"):
        hs, rs, gs = [], [], []
        for i, n in enumerate(sizes):
            h, r = orc.split(fmt, synth.weights(n, 0.02, 40 + i))
            hs.append(h); rs.append(r); gs.append(synth.grads(n, 5e-2, fmt, 41, i))
        V = [dev16(h, fmt) for h in hs]
        R = [torch.from_numpy(r.copy()).cuda() for r in rs]
        G = [dev16(g, fmt) for g in gs]
        M = [torch.zeros(n, device="cuda") for n in sizes]
        W = [torch.zeros(n, device="cuda") for n in sizes]
        if kind == "adam":
            hp = mpo.AdamParams(lr=1e-3, weight_decay=0.1, step=1, clip_value=0.03, grad_scale=0.5)
            mpo.mpo_adam_step(mpo.TensorTable(V, R, G, M, W), hp, exact=True)
        else:
            hp = mpo.SgdParams(lr=0.1, momentum=0.9, first_step=True, clip_value=0.03, grad_scale=0.5)
            mpo.mpo_sgd_step(mpo.TensorTable(V, R, G, M, [None] * 3), hp, exact=True)
        for i, n in enumerate(sizes):
            m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
            if kind == "adam":
                orc.adam_step(fmt, fmt, hs[i], rs[i], gs[i], m, v, lr=1e-3, weight_decay=0.1, grad_scale=0.5,
                              clip_value=0.03)
            else:
                orc.sgd_step(fmt, fmt, hs[i], rs[i], gs[i], m, lr=0.1, momentum=0.9, first_step=True,
                             grad_scale=0.5, clip_value=0.03)
            assert np.array_equal(host16(V[i]), hs[i]) and np.array_equal(R[i].cpu().numpy(), rs[i])
    # hook mode == multi-tensor with clip_value
    a, b, oa, ob = _pair(torch.bfloat16, "adam", mpo, lr=1e-3, clip_value=1e-3)
    ob.install_backward_hooks()
    idx = torch.randint(0, 257, (4, 33), device="cuda")
    _loss(a, idx).backward(); oa.step()
    _loss(b, idx).backward()
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert torch.equal(pa.view(torch.int16), pb.view(torch.int16))


def test_skip_nonfinite_multi_tensor(mpo):
    """Loss-scaling found-inf: one Inf anywhere in the table -> nothing updated (value, residual,
    m, v bit-identical); finite grads -> a normal step; the optimizer reports it."""
    torch.manual_seed(5)
    ps = [torch.nn.Parameter(torch.randn(n, device="cuda") * 0.02) for n in (5000, 77, 4096)]
    for kind in ("adam", "sgd"):
        qs = [torch.nn.Parameter(p.detach().clone()) for p in ps]
        opt = (mpo.ResidualAdamW(qs, lr=1e-3, fmt=torch.float16, skip_nonfinite=True, grad_scale=1 / 1024)
               if kind == "adam" else
               mpo.ResidualSGD(qs, lr=0.1, momentum=0.9, fmt=torch.float16, skip_nonfinite=True))
        for q in qs:
            q.grad = torch.randn_like(q) * 1e-2
        qs[1].grad[3] = float("inf")
        before = [(q.detach().clone(), opt.state[q]["resid"].clone()) for q in qs]
        opt.step()
        assert opt.found_inf()
        for q, (v0, r0) in zip(qs, before):
            assert torch.equal(q.view(torch.int16), v0.view(torch.int16)) and torch.equal(opt.state[q]["resid"], r0)
            if opt.state[q].get("m") is not None:
                assert not opt.state[q]["m"].any()
        qs[1].grad[3] = 0.0
        opt.step()
        assert not opt.found_inf()
        assert any(not torch.equal(q.view(torch.int16), v0.view(torch.int16)) for q, (v0, _) in zip(qs, before))


def test_skip_nonfinite_hook_mode_per_parameter(mpo):
    """Hook mode can only skip the offending parameter; found_inf() reports it."""
    torch.manual_seed(6)
    d = 64
    model = nn.Sequential(nn.Linear(d, d), nn.Linear(d, d)).cuda()
    opt = mpo.ResidualAdamW(model.parameters(), lr=1e-3, fmt=torch.float16, skip_nonfinite=True)
    opt.install_backward_hooks()
    w0 = [p.detach().clone() for p in model.parameters()]
    x = torch.randn(8, d, device="cuda", dtype=torch.float16)
    model[0].weight.register_hook(lambda g: g.index_fill(0, torch.tensor([0], device=g.device), float("inf")))
    model(x).float().sum().backward()
    assert opt.found_inf()
    changed = [not torch.equal(p.view(torch.int16), w.view(torch.int16)) for p, w in zip(model.parameters(), w0)]
    assert changed == [False, True, True, True]     # only layer 0's weight skipped
    assert not opt.found_inf()                       # reset


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_bucketed_hook_sharding_equals_two_phase(mpo, nccl1, kind):
    """Hook mode x sharding: bucket steps issued from the hooks on a side stream
    == the two-phase sharded step, bitwise (world 1)."""
    torch.manual_seed(11)
    mk = lambda: nn.Sequential(nn.Linear(48, 96), nn.GELU(), nn.Linear(96, 48), nn.Linear(48, 10)).cuda()
    a, b = mk(), mk()
    b.load_state_dict(a.state_dict())
    hp = (lambda: mpo.AdamParams(lr=1e-3, weight_decay=0.1)) if kind == "adam" else \
        (lambda: mpo.SgdParams(lr=0.05, momentum=0.9))
    ref = mpo.ShardedResidualOptimizer(list(a.parameters()), kind=kind, fmt=torch.bfloat16, hp=hp())
    bk = mpo.BucketedShardedOptimizer(list(b.parameters()), kind=kind, fmt=torch.bfloat16, hp=hp(), bucket_elems=2048)
    assert len(bk.layout.buckets) > 1
    for t in range(3):
        x = torch.randn(16, 48, device="cuda", dtype=torch.bfloat16)
        ref.zero_grad()
        a(x).float().square().mean().backward()
        ref.step()
        bk.wait()
        b(x).float().square().mean().backward()
        bk.wait()
        for pa, pb in zip(a.parameters(), b.parameters()):
            assert torch.equal(pa.view(torch.int16), pb.view(torch.int16))
    assert bk.step_count == 3
    bk.remove_hooks()


def test_bucketed_sr_streams_per_bucket(mpo, orc, nccl1):
    """Stochastic rounding in the bucketed hook x sharding path: bucket b of rank r draws from stream
    r + world*b (R18), so no two buckets of a step repeat the same draws.  World 1, fp16 SR,
    Adam; the gradient of every parameter is a known constant (loss = sum(p * C_p)), so the oracle
    can step each bucket of the flat buffers with its own stream: bit-exact."""
    from paper_2309_12381_b200 import api
    torch.manual_seed(12)
    shapes = [(40, 24), (24,), (24, 48), (48,), (300,)]
    ps = [nn.Parameter(torch.randn(s, device="cuda") * 0.05) for s in shapes]
    w0 = [p.detach().clone() for p in ps]
    C = [(torch.randn(s, device="cuda") * 1e-2).to(torch.float16) for s in shapes]
    hp = mpo.AdamParams(lr=1e-3, weight_decay=0.0)
    bk = mpo.BucketedShardedOptimizer(ps, kind="adam", fmt=torch.float16, hp=hp, bucket_elems=1024, scheme="sr",
                                      seed=5, exact=True)
    L = bk.layout
    assert len(L.buckets) > 1
    sum(((p * c).float().sum() for p, c in zip(ps, C))).backward()
    bk.wait()
    torch.cuda.synchronize()
    # oracle: the same flat fp32 source split with stream 0, then each bucket stepped with stream b
    src = np.zeros(L.total, np.float32)
    g = np.zeros(L.total, np.uint16)
    for w, c, o in zip(w0, C, L.offsets):
        src[o:o + w.numel()] = w.reshape(-1).cpu().numpy()
        g[o:o + c.numel()] = c.reshape(-1).view(torch.int16).cpu().numpy().view(np.uint16)
    h, r = orc.split_s("sr", "fp16", src, seed=api.step_seed(5, 0), stream=0)
    for b, (o, length, _) in enumerate(L.buckets):
        sl = slice(o, o + length)
        hh, rr = h[sl].copy(), r[sl].copy()
        m = np.zeros(length, np.float32); v = np.zeros(length, np.float32)
        orc.adam_step_s("sr", "fp16", "fp16", hh, rr, g[sl].copy(), m, v, lr=1e-3, weight_decay=0.0, step=1,
                        seed=api.step_seed(5, 1), stream=b)
        assert np.array_equal(bk.value[sl].view(torch.int16).cpu().numpy().view(np.uint16), hh), b
        po = L.part_offsets[b]
        assert np.array_equal(bk.resid[po:po + length].cpu().numpy(), rr), b
    bk.remove_hooks()


def _cudart():
    import ctypes
    import glob
    import nvidia
    for d in nvidia.__path__:
        for f in glob.glob(os.path.join(d, "cuda_runtime", "lib", "libcudart.so*")):
            lib = ctypes.CDLL(f)
            lib.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
            return lib
    raise RuntimeError("libcudart not found")


@pytest.mark.parametrize("kind,fmt", [("adam", "bf16"), ("sgd", "fp16")])
def test_nvls_fused_step_world1_matches_oracle(mpo, orc, kind, fmt):
    """SURVEY 8(f) row 1 at world 1: the fused NVLS kernel (multimem.ld_reduce of the grads,
    multimem.st of the values through a real single-device multicast object) == the oracle step
    bit-exactly (exact build)."""
    from paper_2309_12381_b200 import api
    from paper_2309_12381_b200._lib import MPO_ADAM, MPO_SGD
    from gpu_util import TDT
    rt = _cudart()
    n = 3 * 4096 + 24
    w = synth.weights(n, 0.02, 99)
    h, r = orc.split(fmt, w)
    g = synth.grads(n, 1e-2, fmt, 99, 1)
    try:
        vbuf = api.NvlsLocalBuffer(n * 2, exact=True)
    except mpo.MpoError as e:   # a one-GPU box may refuse a one-device multicast team
        pytest.skip(f"no multicast object on this box: {e}")
    gbuf = api.NvlsLocalBuffer(n * 2, exact=True)
    try:
        hh, gg = np.ascontiguousarray(h), np.ascontiguousarray(g)
        assert rt.cudaMemcpy(vbuf.uc, hh.ctypes.data, n * 2, 1) == 0        # host -> device
        assert rt.cudaMemcpy(gbuf.uc, gg.ctypes.data, n * 2, 1) == 0
        R = torch.from_numpy(r.copy()).cuda()
        M = torch.zeros(n, device="cuda"); V = torch.zeros(n, device="cuda")
        m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
        if kind == "adam":
            hp = mpo.AdamParams(lr=1e-3, weight_decay=0.1, step=1)
            api.mpo_nvls_sharded_step(MPO_ADAM, 0, 1, api.dtype_code(TDT[fmt]), vbuf.mc, vbuf.uc, gbuf.mc, R, M, V,
                                      n, hp, exact=True)
            orc.adam_step(fmt, fmt, h, r, g, m, v, lr=1e-3, weight_decay=0.1, step=1)
        else:
            hp = mpo.SgdParams(lr=0.1, momentum=0.9, first_step=True)
            api.mpo_nvls_sharded_step(MPO_SGD, 0, 1, api.dtype_code(TDT[fmt]), vbuf.mc, vbuf.uc, gbuf.mc, R, M, None,
                                      n, hp, exact=True)
            orc.sgd_step(fmt, fmt, h, r, g, m, lr=0.1, momentum=0.9, first_step=True)
        torch.cuda.synchronize()
        out = np.empty(n, np.uint16)
        assert rt.cudaMemcpy(out.ctypes.data, vbuf.uc, n * 2, 2) == 0        # device -> host
        assert np.array_equal(out, h)
        assert np.array_equal(R.cpu().numpy(), r)
        assert np.array_equal(M.cpu().numpy().view(np.uint32), m.view(np.uint32))
    finally:
        vbuf.free()
        gbuf.free()


def test_hook_mode_optimizer_is_collectable(mpo):
    """Hooks hold the optimizer weakly: dropping the model and the optimizer frees all their
    device memory (no uncollectable hook <-> optimizer cycle)."""
    import gc
    import weakref
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()

    def make():
        m = nn.Sequential(nn.Linear(256, 256), nn.LayerNorm(256)).cuda()
        o = mpo.ResidualAdamW(m.parameters(), lr=1e-3, fmt=torch.bfloat16)
        o.install_backward_hooks()
        m(torch.randn(4, 256, device="cuda", dtype=torch.bfloat16)).float().sum().backward()
        return weakref.ref(o)
    ref = make()
    gc.collect()
    torch.cuda.synchronize()
    assert ref() is None
    assert torch.cuda.memory_allocated() - base < 1 << 16


def _kw_adam(hp):
    return dict(lr=hp.lr, beta1=hp.beta1, beta2=hp.beta2, eps=hp.eps, weight_decay=hp.weight_decay,
                adamw=hp.adamw, grad_scale=hp.grad_scale, step=hp.step)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("kind,fmt,scheme", [("adam", "bf16", "rne"), ("sgd", "fp16", "rne"),
                                             ("adam", "fp16", "sr"), ("adam", "bf16", "x8"), ("sgd", "fp16", "x8z"),
                                             ("adam", "bf16", "rtz")])
def test_p2p_fused_sharded_step_emulated_peers(mpo, orc, world, kind, fmt, scheme, p2p_kernel):
    """SURVEY 8(f) row 1, P2P form: `world` ranks emulated on one device (each with its own
    gradient buffer and value replica; the kernel of rank r reads every rank's gradient shard r
    and writes its new values into every replica).  After all ranks stepped, every replica and
    every shard's residual / m / v equal the oracle: reduce_sum16 (R15) of the ranks' gradients,
    then the oracle step of the shard with grad_scale 1/world (exact build, bit-exact)."""
    from paper_2309_12381_b200 import api
    from paper_2309_12381_b200._lib import MPO_ADAM, MPO_SGD
    from gpu_util import TDT
    S = 8 * (3 * 4096 // 8 + 5)                 # shard: several units past a ragged thread count
    n = S * world
    w = synth.weights(n, 0.02, 7)
    for k in range(world):                       # special values in every shard (slow unit paths)
        w[k * S:k * S + 36] = synth.edge_f32() * np.float32(1e-3)
        w[k * S + 36:k * S + 72] = synth.edge_f32()      # unscaled: overflow, Inf, NaN, max-finite
    h, r = orc.split_s(scheme, fmt, w, seed=3, stream=0)
    gs = [synth.grads(n, 1e-2, fmt, 0xC0FFEE, k) for k in range(world)]
    if world > 1:                                # a non-finite gradient on one rank only
        gs[1][S * (world - 1) + 40] = 0x7C00 if fmt == "fp16" else 0x7F80
    rdt = {"x8": torch.int8, "x8z": torch.uint8}.get(scheme, torch.int16)
    tdt = TDT[fmt]
    V = [torch.from_numpy(h.view(np.int16).copy()).view(tdt).cuda() for _ in range(world)]   # replicas
    G = [torch.from_numpy(g.view(np.int16).copy()).view(tdt).cuda() for g in gs]
    Rs, Ms, Ws = [], [], []
    ms = [synth.normal_f32(S, 1e-3, 5, k) for k in range(world)]
    vs = [np.abs(synth.normal_f32(S, 1e-5, 6, k)) for k in range(world)]
    for k in range(world):
        rk = r[k * S:(k + 1) * S].copy()
        Rs.append(torch.from_numpy(rk if scheme in ("x8", "x8z") else rk.view(np.int16)).cuda().view(rdt))
        Ms.append(torch.from_numpy(ms[k].copy()).cuda())
        Ws.append(torch.from_numpy(vs[k].copy()).cuda())
    seed = 1234
    if kind == "adam":
        hp = mpo.AdamParams(lr=1e-3, weight_decay=0.1, step=4, grad_scale=1.0 / world, seed=seed)
    else:
        hp = mpo.SgdParams(lr=0.1, momentum=0.9, weight_decay=1e-4, grad_scale=1.0 / world, seed=seed)
    vp = [t.data_ptr() for t in V]
    gp = [t.data_ptr() for t in G]
    for k in range(world):
        api.mpo_p2p_sharded_step(MPO_ADAM if kind == "adam" else MPO_SGD, k, world, vp, gp, Rs[k], Ms[k],
                                 Ws[k] if kind == "adam" else None, n, hp, tdt, exact=True, scheme=scheme)
    torch.cuda.synchronize()
    for k in range(world):
        sl = slice(k * S, (k + 1) * S)
        gsum = orc.reduce_sum16(fmt, [g[sl] for g in gs])
        hk, rk = h[sl].copy(), r[sl].copy()
        if kind == "adam":
            orc.adam_step_s(scheme, fmt, "fp32", hk, rk, gsum, ms[k], vs[k], seed=seed, stream=k, **_kw_adam(hp))
        else:
            orc.sgd_step_s(scheme, fmt, "fp32", hk, rk, gsum, ms[k], lr=hp.lr, momentum=hp.momentum,
                           weight_decay=hp.weight_decay, grad_scale=hp.grad_scale, seed=seed, stream=k)
        for rep in V:
            assert np.array_equal(host16(rep)[sl], hk), (k, "value replica")
        got_r = Rs[k].cpu().numpy()
        assert np.array_equal(got_r.view(rk.dtype) if scheme not in ("x8", "x8z") else got_r, rk), (k, "residual")
        assert same_bits_nan_equal(Ms[k].cpu().numpy(), ms[k]), (k, "m")
        if kind == "adam":
            assert same_bits_nan_equal(Ws[k].cpu().numpy(), vs[k]), (k, "v")
    assert all(np.array_equal(host16(G[k]), gs[k]) for k in range(world))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("kind,fmt,scheme", [("adam", "bf16", "rne"), ("sgd", "fp16", "rne"), ("adam", "fp16", "rne"),
                                             ("adam", "fp16", "sr"), ("adam", "bf16", "x8"), ("sgd", "fp16", "x8z"),
                                             ("adam", "bf16", "rtz")])
def test_nvls_kernel_emulated_multicast(mpo, orc, world, kind, fmt, scheme):
    """SURVEY 8(f) row 1, NVLS form, on a box without a multicast object: the NVLS kernel with
    multimem.ld_reduce / multimem.st emulated over `world` ranks' buffers on one device (include/
    mpo.h mpo_nvls_emulated_step).  The emulated reduction is the fp32 sum in rank order rounded
    once to 16 bits -- the oracle's cast16(reduce_sum16(...)) -- then the oracle step of the shard
    with the 16-bit sum as gradient and grad_scale 1/world: every replica and every shard's
    residual / m / v bit-exact (exact build).  Edge weights (overflow, Inf, NaN, max-finite) and a
    non-finite gradient on one rank are in the inputs."""
    from paper_2309_12381_b200 import api
    from paper_2309_12381_b200._lib import MPO_ADAM, MPO_SGD
    from gpu_util import TDT
    S = 8 * (3 * 4096 // 8 + 5)
    n = S * world
    w = synth.weights(n, 0.02, 11)
    for k in range(world):
        w[k * S:k * S + 36] = synth.edge_f32() * np.float32(1e-3)
        w[k * S + 36:k * S + 72] = synth.edge_f32()
    h, r = orc.split_s(scheme, fmt, w, seed=3, stream=0)
    gs = [synth.grads(n, 1e-2, fmt, 0xC0FFEE, 10 + k) for k in range(world)]
    if world > 1:
        gs[1][S * (world - 1) + 40] = 0x7C00 if fmt == "fp16" else 0x7F80
    tdt = TDT[fmt]
    rdt = {"x8": torch.int8, "x8z": torch.uint8}.get(scheme, torch.int16)
    V = [torch.from_numpy(h.view(np.int16).copy()).view(tdt).cuda() for _ in range(world)]
    G = [torch.from_numpy(g.view(np.int16).copy()).view(tdt).cuda() for g in gs]
    ms = [synth.normal_f32(S, 1e-3, 15, k) for k in range(world)]
    vs = [np.abs(synth.normal_f32(S, 1e-5, 16, k)) for k in range(world)]
    Rs = [torch.from_numpy(r[k * S:(k + 1) * S].copy() if scheme in ("x8", "x8z") else
                           r[k * S:(k + 1) * S].view(np.int16).copy()).cuda().view(rdt) for k in range(world)]
    Ms = [torch.from_numpy(x.copy()).cuda() for x in ms]
    Ws = [torch.from_numpy(x.copy()).cuda() for x in vs]
    seed = 4321
    if kind == "adam":
        hp = mpo.AdamParams(lr=1e-3, weight_decay=0.1, step=3, grad_scale=1.0 / world, seed=seed)
    else:
        hp = mpo.SgdParams(lr=0.1, momentum=0.9, weight_decay=1e-4, grad_scale=1.0 / world, seed=seed)
    vp = [t.data_ptr() for t in V]
    gp = [t.data_ptr() for t in G]
    for k in range(world):
        api.mpo_nvls_emulated_step(MPO_ADAM if kind == "adam" else MPO_SGD, k, world, vp, gp, Rs[k], Ms[k],
                                   Ws[k] if kind == "adam" else None, n, hp, tdt, exact=True, scheme=scheme)
    torch.cuda.synchronize()
    for k in range(world):
        sl = slice(k * S, (k + 1) * S)
        g16 = orc.cast16(fmt, orc.reduce_sum16(fmt, [g[sl] for g in gs]))
        hk, rk = h[sl].copy(), r[sl].copy()
        if kind == "adam":     # SR draws: stream = rank, index inside the shard (as the sharded step)
            orc.adam_step_s(scheme, fmt, fmt, hk, rk, g16, ms[k], vs[k], seed=seed, stream=k, **_kw_adam(hp))
        else:
            orc.sgd_step_s(scheme, fmt, fmt, hk, rk, g16, ms[k], lr=hp.lr, momentum=hp.momentum,
                           weight_decay=hp.weight_decay, grad_scale=hp.grad_scale, seed=seed, stream=k)
        for rep in V:
            assert np.array_equal(host16(rep)[sl], hk), (k, "value replica")
        got_r = Rs[k].cpu().numpy()
        assert np.array_equal(got_r.view(rk.dtype) if scheme not in ("x8", "x8z") else got_r, rk), (k, "residual")
        assert same_bits_nan_equal(Ms[k].cpu().numpy(), ms[k]), (k, "m")
        if kind == "adam":
            assert same_bits_nan_equal(Ws[k].cpu().numpy(), vs[k]), (k, "v")
    assert all(np.array_equal(host16(G[k]), gs[k]) for k in range(world))


def test_nvls_emulated_step_rejects(mpo):
    from paper_2309_12381_b200 import api
    from paper_2309_12381_b200._lib import MPO_ADAM
    n = 64
    v = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    g = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    R = torch.zeros(n, dtype=torch.int16, device="cuda")
    M = torch.zeros(n, device="cuda"); W = torch.zeros(n, device="cuda")
    with pytest.raises(mpo.MpoError, match="pre-pass"):
        api.mpo_nvls_emulated_step(MPO_ADAM, 0, 1, [v.data_ptr()], [g.data_ptr()], R, M, W, n,
                                   mpo.AdamParams(lr=1e-3, max_grad_norm=1.0), torch.bfloat16)
    with pytest.raises(mpo.MpoError, match="world"):
        api.mpo_nvls_emulated_step(MPO_ADAM, 0, 9, [v.data_ptr()] * 9, [g.data_ptr()] * 9, R, M, W, 72 * 9,
                                   mpo.AdamParams(lr=1e-3), torch.bfloat16)
    import ctypes as C
    from paper_2309_12381_b200 import _lib
    L = api._lib_of(True)
    arr = (C.c_void_p * 1)(C.c_void_p(v.data_ptr()))
    garr = (C.c_void_p * 1)(C.c_void_p(g.data_ptr()))
    chp = mpo.AdamParams(lr=1e-3).c()
    st = L.mpo_nvls_emulated_step(MPO_ADAM, 0, 1, 99, arr, garr, R.data_ptr(), M.data_ptr(), W.data_ptr(), n,
                                  C.byref(chp), None)
    assert st == _lib.MPO_EDTYPE and b"unsupported storage format" in L.mpo_last_error()


def test_p2p_fused_sharded_step_rejects(mpo):
    from paper_2309_12381_b200 import api
    from paper_2309_12381_b200._lib import MPO_ADAM
    n = 64
    v = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    g = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    R = torch.zeros(n, dtype=torch.int16, device="cuda")
    M = torch.zeros(n, device="cuda"); W = torch.zeros(n, device="cuda")
    with pytest.raises(mpo.MpoError, match="pre-pass"):
        api.mpo_p2p_sharded_step(MPO_ADAM, 0, 1, [v.data_ptr()], [g.data_ptr()], R, M, W, n,
                                 mpo.AdamParams(lr=1e-3, max_grad_norm=1.0), torch.bfloat16)
    with pytest.raises(mpo.MpoError, match="world"):
        api.mpo_p2p_sharded_step(MPO_ADAM, 0, 9, [v.data_ptr()] * 9, [g.data_ptr()] * 9, R, M, W, 72 * 9,
                                 mpo.AdamParams(lr=1e-3), torch.bfloat16)
    with pytest.raises(mpo.MpoError, match="8\\*world"):
        api.mpo_p2p_sharded_step(MPO_ADAM, 0, 2, [v.data_ptr()] * 2, [g.data_ptr()] * 2, R, M, W, 60,
                                 mpo.AdamParams(lr=1e-3), torch.bfloat16)


@pytest.mark.parametrize("kind", ["adamw", "sgd"])
@pytest.mark.parametrize("fmt", [torch.bfloat16, torch.float16])
def test_residual_adamw_tracks_fp32_master_over_many_steps(mpo, fmt, kind):
    """The paper's claim on the GPU path: a 16-bit model whose optimizer keeps the
    residual follows the fp32-master optimizer.  300 AdamW steps on identical 16-bit gradients:
    ResidualAdamW's reconstructed fp32 weights stay within a few fp32 ulps per step of torch's own
    fp32-master AdamW (an independent implementation; op order may differ, R6/R12), while the
    same AdamW run directly on 16-bit parameters (no residual) drifts orders of magnitude further
    (updates below half a 16-bit ulp are lost)."""
    torch.manual_seed(0)
    shapes = [(256, 256), (256,), (64, 256)]
    w0 = [torch.randn(s, device="cuda") * 0.02 for s in shapes]
    if fmt == torch.float16:
        w0 = [w.to(fmt).float() for w in w0]    # fp16-exact start (avoids the < 2^-16 lossy range, R5)
    ref = [w.clone().requires_grad_() for w in w0]
    ps = [nn.Parameter(w.clone()) for w in w0]
    low = [w.to(fmt).requires_grad_() for w in w0]
    if kind == "adamw":
        kw = dict(lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
        o_ref = torch.optim.AdamW(ref, foreach=False, **kw)
        o_low = torch.optim.AdamW(low, foreach=False, **kw)
        opt = mpo.ResidualAdamW(ps, fmt=fmt, **kw)
    else:   # SGD-momentum (the ResNet-50 recipe's optimizer), small lr
        kw = dict(lr=1e-3, momentum=0.9, weight_decay=2e-4)
        o_ref = torch.optim.SGD(ref, foreach=False, **kw)
        o_low = torch.optim.SGD(low, foreach=False, **kw)
        opt = mpo.ResidualSGD(ps, fmt=fmt, **kw)
    for _ in range(300):
        g = [(torch.randn(s, device="cuda") * 1e-2).to(fmt) for s in shapes]
        for r, x in zip(ref, g):
            r.grad = x.float()
        for p, x in zip(ps, g):
            p.grad = x.clone()
        for q, x in zip(low, g):
            q.grad = x.clone()
        o_ref.step()
        opt.step()
        o_low.step()
    torch.cuda.synchronize()
    w_res = opt.fp32_params()
    err_res = max(float((a.reshape(-1) - r.detach().reshape(-1)).abs().max()) for a, r in zip(w_res, ref))
    # (fp16-only AdamW may even produce NaN: v and eps underflow in fp16 -- infinitely worse)
    err_low = max(float(torch.nan_to_num((q.detach().float() - r.detach()).abs(), nan=float("inf")).max())
                  for q, r in zip(low, ref))
    scale = max(float(r.detach().abs().max()) for r in ref)
    assert err_res <= 300 * 2.0 ** -23 * scale, (err_res, scale)      # <= 1 fp32 ulp of the scale per step
    assert err_low > 100 * err_res, (err_low, err_res)


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_add_param_group(mpo, kind):
    """torch.optim's add_param_group: (a) a group added before the first step gives the same
    steps as passing both groups to the constructor; (b) added after two steps, the first group
    continues exactly as an optimizer over it alone and the new group steps like a fresh optimizer
    over it (its counts start at 0); refused while backward hooks are installed."""
    torch.manual_seed(5)
    A = [torch.randn(300, 17, device="cuda") * 0.02, torch.randn(4100, device="cuda") * 0.02]
    B = [torch.randn(64, 65, device="cuda") * 0.02]
    mk = (lambda groups: mpo.ResidualAdamW(groups, lr=1e-3, weight_decay=0.1, fmt=torch.bfloat16)) \
        if kind == "adam" else (lambda groups: mpo.ResidualSGD(groups, lr=0.1, momentum=0.9, fmt=torch.bfloat16))
    grads = [[(torch.randn(t.shape, device="cuda") * 1e-2).to(torch.bfloat16) for t in A + B] for _ in range(4)]

    def run(opt, ps, steps):
        for t in steps:
            for p, g in zip(ps, grads[t]):
                p.grad = g.clone()
            opt.step()

    pa = [nn.Parameter(t.clone()) for t in A + B]
    oa = mk([{"params": pa[:2]}])
    oa.add_param_group({"params": pa[2:], "lr": 5e-4 if kind == "adam" else 0.05})
    pb = [nn.Parameter(t.clone()) for t in A + B]
    ob = mk([{"params": pb[:2]}, {"params": pb[2:], "lr": 5e-4 if kind == "adam" else 0.05}])
    run(oa, pa, range(4)); run(ob, pb, range(4))
    for x, y in zip(pa, pb):
        assert torch.equal(x.view(torch.int16), y.view(torch.int16))
        assert torch.equal(oa.state[x]["resid"], ob.state[y]["resid"])
    # (b) added after two steps
    pc = [nn.Parameter(t.clone()) for t in A + B]
    oc = mk([{"params": pc[:2]}])
    run(oc, pc[:2], range(2))
    oc.add_param_group({"params": pc[2:]})
    run(oc, pc, range(2, 4))
    pd = [nn.Parameter(t.clone()) for t in A]
    od = mk([{"params": pd}])
    run(od, pd, range(4))
    pe = [nn.Parameter(t.clone()) for t in B]
    oe = mk([{"params": pe}])
    for t in range(2, 4):
        pe[0].grad = grads[t][2].clone()
        oe.step()
    for x, y in zip(pc, pd + pe):
        assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    assert [int(oc.state[p]["step"]) for p in pc] == [4, 4, 2]
    assert set(oc.state_dict()["state"]) == {0, 1, 2}
    oc.install_backward_hooks()
    with pytest.raises(mpo.MpoError, match="add_param_group"):
        oc.add_param_group({"params": [nn.Parameter(torch.zeros(8, device="cuda"))]})


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_more_param_groups_than_one_hp_bank(mpo, kind):
    """Layer-wise lr decay over 20 param groups (> the 16 hyper-parameter groups one launch
    carries): the multi-tensor step, the native and the Python hooks (small parameters batched
    into end-of-backward flushes of 20 (group, step) pairs) all split into launches of <= 16 and
    equal one optimizer per layer, bitwise."""
    torch.manual_seed(11)
    L = 20

    def make():
        torch.manual_seed(11)
        return nn.Sequential(*[nn.Linear(16, 16) for _ in range(L)]).cuda()

    def groups(m):
        return [{"params": list(m[i].parameters()), "lr": (1e-3 if kind == "adam" else 0.1) * 0.9 ** i}
                for i in range(L)]
    mk = (lambda g: mpo.ResidualAdamW(g, lr=1e-3, weight_decay=0.1, fmt=torch.bfloat16)) if kind == "adam" else \
        (lambda g: mpo.ResidualSGD(g, lr=0.1, momentum=0.9, fmt=torch.bfloat16))
    models = [make() for _ in range(4)]
    oa = mk(groups(models[0]))
    ob = mk(groups(models[1])); ob.install_backward_hooks(native=True)
    oc = mk(groups(models[2])); oc.install_backward_hooks(native=False)
    od = [mk([g]) for g in groups(models[3])]
    gen = torch.Generator(device="cuda").manual_seed(12)
    for _ in range(3):
        x = torch.randn(8, 16, device="cuda", dtype=torch.bfloat16, generator=gen)
        for k, m in enumerate(models):
            m(x).float().square().mean().backward()
            if k == 0:
                oa.step()
            elif k == 3:
                for o in od:
                    o.step()
            if k in (0, 3):
                for p in m.parameters():
                    p.grad = None
    for k in (1, 2, 3):
        for pa, pk in zip(models[0].parameters(), models[k].parameters()):
            assert torch.equal(pa.view(torch.int16), pk.view(torch.int16)), k


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_torch_grad_scaler_protocol(mpo, kind):
    """torch.amp.GradScaler drives the residual optimizers through its fused-optimizer protocol
    (`_step_supports_amp_scaling`: it sets optimizer.grad_scale / found_inf before step()): the
    unscale happens inside the step (grad_scale = 1/scale) and equals an optimizer stepped on the
    same scaled gradients with that grad_scale, bitwise; a step with a non-finite scaled gradient
    is skipped (no update, no step count) and the scaler backs off; hook mode refuses it."""
    torch.manual_seed(21)
    a, b = TinyLM().cuda().half(), TinyLM().cuda().half()
    b.load_state_dict(a.state_dict())
    mk = (lambda m: mpo.ResidualAdamW(m.parameters(), lr=1e-3, weight_decay=0.1, fmt=torch.float16)) \
        if kind == "adam" else (lambda m: mpo.ResidualSGD(m.parameters(), lr=0.1, momentum=0.9, fmt=torch.float16))
    oa, ob = mk(a), mk(b)
    scaler = torch.amp.GradScaler("cuda", init_scale=2.0 ** 10, growth_interval=1)
    gen = torch.Generator(device="cuda").manual_seed(22)
    for it in range(4):
        idx = torch.randint(0, 257, (4, 33), device="cuda", generator=gen)
        scale = float(scaler.get_scale())
        scaler.scale(_loss(a, idx)).backward()
        (_loss(b, idx) * torch.full((), scale, device="cuda")).backward()
        if it == 3:                                   # a non-finite scaled gradient
            next(a.parameters()).grad.view(-1)[0] = float("inf")
            before = [p.detach().clone() for p in a.parameters()]
        scaler.step(oa)
        scaler.update()
        if it < 3:
            for g in ob.param_groups:
                g["grad_scale"] = 1.0 / scale
            ob.step()
            for pa, pb in zip(a.parameters(), b.parameters()):
                assert torch.equal(pa.view(torch.int16), pb.view(torch.int16)), it
        else:
            assert all(torch.equal(x, p) for x, p in zip(before, a.parameters()))
            assert all(int(oa.state[p]["step"]) == 3 for p in a.parameters())
            assert float(scaler.get_scale()) == scale / 2
        for m in (a, b):
            for p in m.parameters():
                p.grad = None
    assert "found_inf" not in oa.__dict__ and oa._amp_inv == 1.0   # (found_inf() is also a method)
    oh = mk(b)
    oh.install_backward_hooks()
    scaler2 = torch.amp.GradScaler("cuda")
    scaler2.scale(_loss(b, idx)).backward()
    with pytest.raises(mpo.MpoError, match="GradScaler"):
        scaler2.step(oh)


@pytest.mark.parametrize("native", [True, False])
def test_empty_and_frozen_parameters(mpo, native):
    """Zero-element parameters and parameters without gradients ride along: the multi-tensor step
    and both hook modes skip them and step the rest exactly as without them."""
    torch.manual_seed(41)
    ref = [torch.randn(300, device="cuda") * 0.02, torch.randn(17, 5, device="cuda") * 0.02]
    pa = [nn.Parameter(t.clone()) for t in ref]
    pb = [nn.Parameter(t.clone()) for t in ref] + [nn.Parameter(torch.empty(0, device="cuda")),
                                                   nn.Parameter(torch.randn(8, device="cuda"), requires_grad=False)]
    oa = mpo.ResidualAdamW(pa, lr=1e-3, fmt=torch.bfloat16)
    ob = mpo.ResidualAdamW(pb, lr=1e-3, fmt=torch.bfloat16)
    oc_params = [nn.Parameter(t.clone()) for t in ref] + [nn.Parameter(torch.empty(0, device="cuda"))]
    oc = mpo.ResidualAdamW(oc_params, lr=1e-3, fmt=torch.bfloat16)
    oc.install_backward_hooks(native=native, batch_below=0)
    frozen = pb[3].detach().clone()
    x = torch.randn(300, device="cuda", dtype=torch.bfloat16)
    y = torch.randn(17, 5, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        for ps, o in ((pa, oa), (pb, ob), (oc_params, oc)):
            loss = (ps[0] * x).float().sum() + (ps[1] * y).float().square().sum()
            if len(ps) > 2:
                loss = loss + ps[2].float().sum()
            loss.backward()
            if o is not oc:
                o.step()
                for p in ps:
                    p.grad = None
    for i in range(2):
        assert torch.equal(pa[i].view(torch.int16), pb[i].view(torch.int16))
        assert torch.equal(pa[i].view(torch.int16), oc_params[i].view(torch.int16))
    assert torch.equal(pb[3], frozen) and pb[2].numel() == 0
