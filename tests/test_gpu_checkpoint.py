"""GPU: optimizer checkpoint / resume, the step counts of skipped (found-inf) updates, and one
global-norm pre-pass over every table of a step.

* "Extra bits are stored by the optimizer": the residual is optimizer state, so a resumed
  run must continue bit-identically.  Train 3 steps -> torch.save(model, optimizer) -> a FRESH
  model + optimizer -> load both -> 3 more steps == 6 uninterrupted steps, bitwise (values,
  residuals, m, v, step counts), for multi-tensor and hook mode, bf16 and fp16, RNE and stochastic
  rounding (whose draws are keyed by the step count and the per-parameter stream).
* A skipped update (loss-scaling found-inf) does not advance the bias-correction step
  count (torch's GradScaler never calls the optimizer's step then).
* Global-norm clipping over parameters whose gradients have different dtypes (several launches)
  uses ONE norm over all of them (R9).
"""
import io

import numpy as np
import pytest
import torch
import torch.nn as nn

import synth
from gpu_util import dev16, dev_grad, host16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_12381_b200 as m
    from paper_2309_12381_b200 import _build
    _build.build()
    return m


class Net(nn.Module):
    def __init__(self, d=48, vocab=101):
        super().__init__()
        self.emb = nn.Embedding(vocab, d)
        self.ln = nn.LayerNorm(d)
        self.fc1 = nn.Linear(d, 3 * d)
        self.fc2 = nn.Linear(3 * d, d)

    def forward(self, idx):
        x = self.emb(idx)
        x = x + self.fc2(torch.nn.functional.gelu(self.fc1(self.ln(x))))
        return x @ self.emb.weight.t()


def _loss(model, idx):
    logits = model(idx[:, :-1]).float()
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), idx[:, 1:].reshape(-1))


def _make(mpo, kind, fmt, scheme, seed_init, hook):
    torch.manual_seed(seed_init)
    model = Net().cuda()
    if kind == "adam":
        opt = mpo.ResidualAdamW(model.parameters(), lr=2e-3, betas=(0.9, 0.95), weight_decay=0.1, fmt=fmt,
                                scheme=scheme, seed=11, exact=True)
    else:
        opt = mpo.ResidualSGD(model.parameters(), lr=0.05, momentum=0.9, weight_decay=1e-4, fmt=fmt, scheme=scheme,
                              seed=11, exact=True)
    if hook:
        opt.install_backward_hooks()
    return model, opt


def _train(model, opt, steps, hook, start):
    for t in range(start, start + steps):
        gen = torch.Generator(device="cuda").manual_seed(1000 + t)
        idx = torch.randint(0, 101, (4, 17), device="cuda", generator=gen)
        _loss(model, idx).backward()
        if not hook:
            opt.step()
            for p in model.parameters():
                p.grad = None


def _snapshot(model, opt):
    out = []
    for p in model.parameters():
        st = opt.state[p]
        out.append((p.detach().view(torch.int16).clone(), st["resid"].clone(), st["step"],
                    None if st.get("m") is None else st["m"].clone(), None if st.get("v") is None else st["v"].clone()))
    return out


@pytest.mark.parametrize("kind", ["adam", "sgd"])
@pytest.mark.parametrize("fmt,scheme", [(torch.bfloat16, "rne"), (torch.float16, "rne"), (torch.float16, "sr"),
                                        (torch.bfloat16, "x8z")])
@pytest.mark.parametrize("hook", [False, True])
def test_resume_is_bit_identical(mpo, kind, fmt, scheme, hook):
    a, oa = _make(mpo, kind, fmt, scheme, 0, hook)
    _train(a, oa, 6, hook, 0)
    ref = _snapshot(a, oa)

    b, ob = _make(mpo, kind, fmt, scheme, 0, hook)
    _train(b, ob, 3, hook, 0)
    buf = io.BytesIO()
    torch.save({"model": b.state_dict(), "opt": ob.state_dict()}, buf)
    del b, ob
    buf.seek(0)
    ck = torch.load(buf, weights_only=False)
    # the saved state keeps its own dtypes: fp32 moments, integer residual codes, int steps
    for st in ck["opt"]["state"].values():
        assert st["resid"].dtype == mpo.api.resid_dtype(scheme) and isinstance(st["step"], int) and st["step"] == 3
        for k in ("m", "v"):
            if st.get(k) is not None:
                assert st[k].dtype == torch.float32
    c, oc = _make(mpo, kind, fmt, scheme, 1234, hook)     # different init: everything must come from the file
    c.load_state_dict(ck["model"])
    oc.load_state_dict(ck["opt"])
    _train(c, oc, 3, hook, 3)
    got = _snapshot(c, oc)
    for (pa, ra, sa, ma, va), (pc, rc, sc, mc, vc) in zip(ref, got):
        assert torch.equal(pa, pc) and torch.equal(ra, rc) and sa == sc == 6
        for x, y in ((ma, mc), (va, vc)):
            assert (x is None) == (y is None)
            if x is not None:
                assert torch.equal(x.view(torch.int32), y.view(torch.int32))


def test_load_state_dict_rejects_mismatch(mpo):
    a, oa = _make(mpo, "adam", torch.bfloat16, "rne", 0, False)
    sd = oa.state_dict()
    b, ob = _make(mpo, "sgd", torch.bfloat16, "rne", 0, False)
    with pytest.raises(mpo.MpoError):
        ob.load_state_dict(sd)
    c, oc = _make(mpo, "adam", torch.float16, "sr", 0, False)
    with pytest.raises(mpo.MpoError):
        oc.load_state_dict(sd)
    bad = {**sd, "state": {k: {**v, "m": v["m"].to(torch.bfloat16)} for k, v in sd["state"].items()}}
    a2, oa2 = _make(mpo, "adam", torch.bfloat16, "rne", 0, False)
    with pytest.raises(mpo.MpoError, match="float32"):
        oa2.load_state_dict(bad)
    with pytest.raises(mpo.MpoError):
        oa2.load_state_dict({"state": {}, "param_groups": sd["param_groups"]})


@pytest.mark.parametrize("kind", ["adam", "sgd"])
def test_skipped_step_does_not_count(mpo, kind):
    """Multi-tensor: an Inf gradient skips the update AND its step count: the next finite step is
    bit-identical to the first step of an optimizer that never saw the skipped one."""
    torch.manual_seed(3)
    ps = [torch.randn(n, device="cuda") * 0.02 for n in (5000, 77, 4096)]

    def mk():
        qs = [nn.Parameter(p.clone()) for p in ps]
        if kind == "adam":
            return qs, mpo.ResidualAdamW(qs, lr=1e-3, fmt=torch.float16, skip_nonfinite=True, exact=True)
        return qs, mpo.ResidualSGD(qs, lr=0.1, momentum=0.9, fmt=torch.float16, skip_nonfinite=True, exact=True)
    qa, oa = mk()
    qb, ob = mk()
    g = [(torch.randn_like(p) * 1e-2).to(torch.float16) for p in ps]
    for q in qa:
        q.grad = torch.randn_like(q)
    qa[2].grad[7] = float("inf")
    oa.step()                                 # skipped
    for q, gg in zip(qa, g):
        q.grad = gg.clone()
    oa.step()                                 # its first real step
    for q, gg in zip(qb, g):
        q.grad = gg.clone()
    ob.step()
    for x, y in zip(qa, qb):
        assert torch.equal(x.view(torch.int16), y.view(torch.int16))
        assert oa.state[x]["step"] == ob.state[y]["step"] == 1
        assert torch.equal(oa.state[x]["m"], ob.state[y]["m"])


def test_skipped_hook_step_does_not_count(mpo):
    """Hook mode skips per parameter: only the offending parameter's count stays behind."""
    torch.manual_seed(6)
    d = 64
    model = nn.Sequential(nn.Linear(d, d), nn.Linear(d, d)).cuda()
    opt = mpo.ResidualAdamW(model.parameters(), lr=1e-3, fmt=torch.float16, skip_nonfinite=True)
    opt.install_backward_hooks()
    x = torch.randn(8, d, device="cuda", dtype=torch.float16)
    h = model[0].weight.register_hook(lambda g: g.index_fill(0, torch.tensor([0], device=g.device), float("inf")))
    model(x).float().sum().backward()
    h.remove()
    model(x).float().sum().backward()
    steps = [st["step"] for st in opt.state_dict()["state"].values()]
    assert steps == [1, 2, 2, 2]


@pytest.mark.parametrize("clip", [True, False])
def test_global_norm_over_gradient_dtypes(mpo, orc, clip):
    """Two parameters whose gradients differ in dtype (fp16 and fp32: two launches) share ONE norm:
    S on the device equals the oracle's S over both (1e-10), and the clipped step equals the oracle
    stepped with that coefficient (hybrid, exact build).  With skip_nonfinite, an Inf in the fp32
    gradient also stops the fp16-gradient launch."""
    fmt = "fp16"
    sizes = (9000, 4101)
    ws_ = [synth.weights(n, 0.02, 40 + i) for i, n in enumerate(sizes)]
    ps = [nn.Parameter(torch.from_numpy(w.copy()).cuda()) for w in ws_]
    if clip:
        opt = mpo.ResidualAdamW(ps, lr=1e-3, fmt=torch.float16, max_grad_norm=0.05, exact=True)
    else:
        opt = mpo.ResidualAdamW(ps, lr=1e-3, fmt=torch.float16, skip_nonfinite=True, exact=True)
    hs, rs = zip(*[orc.split(fmt, w) for w in ws_])
    hs, rs = [h.copy() for h in hs], [r.copy() for r in rs]
    g0 = synth.grads(sizes[0], 1e-2, "fp16", 5, 0)
    g1 = synth.grads(sizes[1], 1e-2, "fp32", 5, 1)
    if not clip:
        g1[5] = np.inf
    ps[0].grad = dev_grad(g0, "fp16")
    ps[1].grad_dtype = None          # an fp32 gradient on an fp16 parameter (torch checks by default)
    ps[1].grad = dev_grad(g1, "fp32")
    before = [p.detach().clone() for p in ps]
    opt.step()
    torch.cuda.synchronize()
    S = float(opt._norm_ws[0].item())
    if not clip:
        assert not np.isfinite(S)
        for p, b in zip(ps, before):
            assert torch.equal(p.view(torch.int16), b.view(torch.int16))
        return
    S_orc = orc.sumsq("fp16", g0) + orc.sumsq("fp32", g1)
    assert abs(S - S_orc) <= 1e-10 * S_orc
    coef = orc.clip_coef(S, 0.05)
    assert coef < 1.0
    for i, (g, gf) in enumerate(((g0, "fp16"), (g1, "fp32"))):
        m = np.zeros(sizes[i], np.float32); v = np.zeros(sizes[i], np.float32)
        orc.adam_step(fmt, gf, hs[i], rs[i], g, m, v, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                      adamw=True, step=1, clip_coef=coef)
        assert np.array_equal(host16(ps[i]), hs[i])
        assert np.array_equal(opt.state[ps[i]]["resid"].cpu().numpy(), rs[i])
