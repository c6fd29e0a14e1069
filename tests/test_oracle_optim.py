"""Pins of the oracle's optimizer steps, clipping and byte model (no GPU).

* P5  absorption: the split storage follows a plain numpy
      binary32 loop bit-exactly while a 16-bit-only parameter never moves.
* P6  fp32-master equivalence with event accounting: the residual-compensated
      trajectory equals the fp32-master trajectory bit-exactly on every element whose split
      was never lossy, and within a stated drift bound on the rest.
* P7  special cases / closed forms (first Adam step).
* P10 library routine: torch.optim.SGD / Adam / AdamW (foreach=False, CPU fp32) reproduce
      the oracle's fp32-master trajectory within a few binary32 ulps.
* norm: exact-sum constructions and math.fsum; clip formula closed forms (reading R9).
* P9  byte model.
"""
import math

import numpy as np
import pytest

import synth


def f32(x):
    return np.float32(x)


# ----------------------------------------------------------------------------------- P5 --
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_p5_absorption_repair(orc, fmt):
    n_steps, inc = 1000, f32(1e-4)
    # plain numpy binary32 sequential accumulation (an fp32 master copy)
    w_ref = f32(1.0)
    for _ in range(n_steps):
        w_ref = f32(w_ref + inc)
    # SPEC S:252 expects "1.1 within 1e-5": the binary32 result is 1.1000166 (rel 1.5e-5)
    assert w_ref.view(np.uint32) == 0x3F8CCD58
    # residual-compensated storage: SGD with lr=1 and grad=-1e-4 (fp32 grad)
    h, r = orc.split(fmt, np.array([1.0], np.float32))
    g = np.array([-inc], np.float32)
    for _ in range(n_steps):
        orc.sgd_step(fmt, "fp32", h, r, g, None, lr=1.0)
    assert orc.reconstruct(fmt, h, r)[0].view(np.uint32) == w_ref.view(np.uint32)
    # 16-bit only: the increment is below half an ulp of 1.0 and is absorbed every time
    h16 = orc.cast16(fmt, np.array([1.0], np.float32))
    for _ in range(n_steps):
        h16 = orc.cast16(fmt, orc.widen(fmt, h16) + inc)
    assert orc.widen(fmt, h16)[0] == 1.0
    # SGD direction: 1000 x (-1e-4) from 1.0
    w_ref = f32(1.0)
    for _ in range(n_steps):
        w_ref = f32(w_ref - inc)
    h, r = orc.split(fmt, np.array([1.0], np.float32))
    for _ in range(n_steps):
        orc.sgd_step(fmt, "fp32", h, r, -g, None, lr=1.0)
    assert orc.reconstruct(fmt, h, r)[0] == w_ref


# ----------------------------------------------------------------------------------- P6 --
def _ulp32(x):
    x = np.abs(x.astype(np.float64))
    e = np.floor(np.log2(np.maximum(x, 2.0 ** -126)))
    return 2.0 ** (e - 23)


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
@pytest.mark.parametrize("seed", [0xB0B, 2023])
def test_p6_master_equivalence_adamw(orc, fmt, seed):
    n, T = 1 << 16, 60
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, adamw=True)
    w0 = synth.weights(n, 0.02, seed)
    # fp32 master trajectory
    wm = w0.copy(); mm = np.zeros(n, np.float32); vm = np.zeros(n, np.float32)
    # residual-compensated trajectory, stepped as reconstruct -> fp32 update -> split so the
    # lossy split events can be counted
    h, r = orc.split(fmt, w0)
    ms = np.zeros(n, np.float32); vs = np.zeros(n, np.float32)
    ev0 = orc.reconstruct(fmt, h, r).view(np.uint32) != w0.view(np.uint32)   # initial split
    k = ev0.astype(np.int64)                  # lossy splits per element
    t_first = np.where(ev0, 0, T + 1)         # step of the first event
    j = (ev0 & (np.abs(w0) < 2.0 ** -17)).astype(np.int64)   # events in fp16's saturated range
    wmax = np.abs(w0).astype(np.float64)
    # check the one-call step equals the composition on a copy
    h1, r1, m1, v1 = h.copy(), r.copy(), ms.copy(), vs.copy()
    for t in range(1, T + 1):
        g = synth.grads(n, 1e-3, fmt, seed, t)
        orc.adam_step_master(fmt, wm, g, mm, vm, step=t, **hp)
        w = orc.reconstruct(fmt, h, r)
        orc.adam_step_master(fmt, w, g, ms, vs, step=t, **hp)
        h, r = orc.split(fmt, w)
        rec = orc.reconstruct(fmt, h, r)
        ev = rec.view(np.uint32) != w.view(np.uint32)
        k += ev
        t_first = np.where(ev & (t_first > T), t, t_first)
        j += (np.abs(w) < 2.0 ** -17) & ev
        wmax = np.maximum(wmax, np.abs(w).astype(np.float64))
        orc.adam_step(fmt, fmt, h1, r1, g, m1, v1, step=t, **hp)
    assert np.array_equal(h1, h) and np.array_equal(r1, r)
    assert np.array_equal(m1, ms) and np.array_equal(v1, vs)
    ws = orc.reconstruct(fmt, h, r)
    diff = ws.view(np.uint32) != wm.view(np.uint32)
    no_event = k == 0
    # zero tolerance where the storage never lost a bit
    assert not (diff & no_event).any()
    assert no_event.mean() > 0.9
    # drift bound for elements with events: each lossy split costs <= 1 ulp32 (or 2^-25 in
    # fp16's saturated range), each later step adds <= 2 independent roundings
    d = np.abs(ws.astype(np.float64) - wm.astype(np.float64))
    bound = (k + 2 * np.maximum(T - t_first, 0)) * _ulp32(wmax) + j * 2.0 ** -25
    assert (d <= bound + 0.0).all(), (d - bound).max()


# ----------------------------------------------------------------------------------- P7 --
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_p7_adam_zero_grad(orc, fmt):
    n = 4096
    w0 = synth.weights(n)
    h, r = orc.split(fmt, w0)
    g = np.zeros(n, np.uint16)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    h0, r0 = h.copy(), r.copy()
    orc.adam_step(fmt, fmt, h, r, g, m, v, lr=1e-3, adamw=False, step=1)
    assert np.array_equal(h, h0) and np.array_equal(r, r0)
    # AdamW with g=0 multiplies by (1 - lr*wd) only
    orc.adam_step(fmt, fmt, h, r, g, m, v, lr=1e-3, weight_decay=0.1, adamw=True, step=2)
    w = orc.reconstruct(fmt, h0, r0)
    expect = (w * f32(1.0 - 1e-3 * 0.1)).astype(np.float32)
    eh, er = orc.split(fmt, expect)
    assert np.array_equal(h, eh) and np.array_equal(r, er)


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_p7_sgd_special_cases(orc, fmt):
    n = 4096
    w0 = synth.weights(n)
    g16 = synth.grads(n, 1e-2, fmt, 0xB0B, 1)
    g = orc.widen(fmt, g16)
    h, r = orc.split(fmt, w0)
    w = orc.reconstruct(fmt, h, r)
    # lr = 0: parameter unchanged, momentum buffer updated; carve-out: -0 - (-0) = +0
    buf = np.zeros(n, np.float32)
    hh, rr = h.copy(), r.copy()
    orc.sgd_step(fmt, fmt, hh, rr, g16, buf, lr=0.0, momentum=0.9, first_step=True)
    assert np.array_equal(hh, h) and np.array_equal(rr, r)
    assert np.array_equal(buf, g)                       # first step: buffer = clone(grad)
    # mu = 0, wd = 0: w - lr*g, compared with numpy binary32 arithmetic
    hh, rr = h.copy(), r.copy()
    orc.sgd_step(fmt, fmt, hh, rr, g16, None, lr=0.5)
    expect = (w - f32(0.5) * g).astype(np.float32)
    eh, er = orc.split(fmt, expect)
    assert np.array_equal(hh, eh) and np.array_equal(rr, er)


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_p7_first_adam_step_moves_by_lr(orc, fmt):
    n = 1 << 14
    w0 = synth.weights(n)
    g16 = synth.grads(n, 1e-3, fmt, 2023, 1)
    g = orc.widen(fmt, g16).astype(np.float64)
    wm = w0.copy()
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    lr, eps = 1e-3, 1e-8
    orc.adam_step_master(fmt, wm, g16, m, v, lr=lr, eps=eps, adamw=False, step=1)
    assert np.array_equal(m, (f32(0.1) * g.astype(np.float32)).astype(np.float32))
    moved = w0.astype(np.float64) - wm.astype(np.float64)
    expect = lr * g / (np.abs(g) + eps)
    tol = 8 * _ulp32(np.maximum(np.abs(w0), np.abs(wm))) + 1e-6 * lr
    assert (np.abs(moved - expect) <= tol).all()


# ---------------------------------------------------------------------------------- P10 --
@pytest.mark.parametrize("kind", ["adamw", "adam_l2", "sgd_m", "sgd_nesterov", "sgd_damp_wd",
                                  "adam_b1_0", "adam_b1_03", "adamw_b1_05"])
def test_p10_matches_torch_optim(orc, kind):
    import torch
    n, T = 8192, 30
    w0 = synth.weights(n, 0.02, 0xC0FFEE)
    p = torch.nn.Parameter(torch.from_numpy(w0.copy()))
    # beta1 <= 0.5 (lerp weight 1-beta1 >= 0.5) drives the oracle's upper lerp branch (reading R6,
    # torch's lerp switches formula at weight 0.5): pinned here against torch.optim too
    upper = {"adam_b1_0": (0.0, 0.999, False), "adam_b1_03": (0.3, 0.99, False), "adamw_b1_05": (0.5, 0.95, True)}
    if kind in upper:
        b1, b2, aw = upper[kind]
        hp = dict(lr=1e-3, beta1=b1, beta2=b2, eps=1e-8, weight_decay=0.05, adamw=aw)
        cls = torch.optim.AdamW if aw else torch.optim.Adam
        opt = cls([p], lr=1e-3, betas=(b1, b2), eps=1e-8, weight_decay=0.05, foreach=False, fused=False)
    elif kind == "adamw":
        hp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, adamw=True)
        opt = torch.optim.AdamW([p], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1,
                                foreach=False, fused=False)
    elif kind == "adam_l2":
        hp = dict(lr=7e-5, beta1=0.64, beta2=0.999, eps=1e-8, weight_decay=1e-2, adamw=False)
        opt = torch.optim.Adam([p], lr=7e-5, betas=(0.64, 0.999), eps=1e-8, weight_decay=1e-2,
                               foreach=False, fused=False)
    elif kind == "sgd_m":
        hp = dict(lr=0.3, momentum=0.9, weight_decay=2e-4)
        opt = torch.optim.SGD([p], lr=0.3, momentum=0.9, weight_decay=2e-4, foreach=False)
    elif kind == "sgd_nesterov":
        hp = dict(lr=0.1, momentum=0.9, nesterov=True)
        opt = torch.optim.SGD([p], lr=0.1, momentum=0.9, nesterov=True, foreach=False)
    else:
        hp = dict(lr=0.1, momentum=0.8, dampening=0.3, weight_decay=1e-3)
        opt = torch.optim.SGD([p], lr=0.1, momentum=0.8, dampening=0.3, weight_decay=1e-3,
                              foreach=False)
    w = w0.copy()
    wmax = np.abs(w0).astype(np.float64)
    a = np.zeros(n, np.float32); b = np.zeros(n, np.float32)
    for t in range(1, T + 1):
        g = synth.grads(n, 1e-2, "fp32", 0xC0FFEE, t)
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        if kind.startswith("adam"):
            orc.adam_step_master("fp32", w, g, a, b, step=t, **hp)
        else:
            orc.sgd_step_master("fp32", w, g, a, first_step=(t == 1), **hp)
        wmax = np.maximum(wmax, np.abs(w))
    ref = p.detach().numpy().astype(np.float64)
    err = np.abs(w.astype(np.float64) - ref)
    # a few binary32 ulps of the weight per step at most (torch's CPU kernels may contract)
    assert (err <= 2 * T * _ulp32(wmax)).all(), err.max()
    assert np.median(err / _ulp32(wmax)) <= 1.0


# ------------------------------------------------------------------------------ norm ------
def test_norm_exact_sum_construction(orc):
    # all |g| equal to one power of two: every partial sum is exact in any order
    n = 100_000
    sign = synth.rng(5, 5).integers(0, 2, size=n).astype(np.float32) * 2 - 1
    g = (sign * f32(2.0 ** -7)).astype(np.float32)
    for fmt in ("fp16", "bf16"):
        g16 = orc.cast16(fmt, g)
        assert orc.sumsq(fmt, g16) == n * 2.0 ** -14
        assert orc.sumsq(fmt, g16, grad_scale=0.5) == n * 2.0 ** -16
    assert orc.sumsq("fp32", g) == n * 2.0 ** -14
    assert orc.sumsq("fp32", np.zeros(0, np.float32)) == 0.0


def test_norm_matches_fsum(orc):
    g = synth.grads(1 << 18, 1.0, "fp32", 2023, 3)
    s = orc.sumsq("fp32", g)
    ref = math.fsum((g.astype(np.float64) ** 2).tolist())
    assert abs(s - ref) <= 1e-15 * ref


def test_clip_coef_closed_forms(orc):
    # coef = min(1, max_norm / (norm + 1e-6))  (torch clip_grad_norm_, reading R9)
    assert orc.clip_coef(4.0, 1.0) == f32(1.0 / (2.0 + 1e-6))
    assert orc.clip_coef(0.25, 1.0) == 1.0
    # torch's formula clips slightly even at norm == max_norm
    assert orc.clip_coef(1.0, 1.0) < 1.0
    assert orc.clip_coef(0.0, 1.0) == 1.0
    assert math.isnan(orc.clip_coef(float("nan"), 1.0))
    assert orc.clip_coef(float("inf"), 1.0) == 0.0


@pytest.mark.parametrize("adamw", [False, True])
def test_clipped_step_matches_torch_clip_grad_norm_and_adam(orc, adamw):
    """Global-norm clipping (R9) pinned against library routines: loss-scaled 16-bit
    gradients of several tensors are unscaled (grad_scale), clipped with
    torch.nn.utils.clip_grad_norm_ over ALL tensors and stepped with torch.optim.Adam/AdamW on an
    fp32 master; the oracle computes S = sum (g*gs)^2 over the tensors, coef = clip_coef(S), and
    steps each tensor with it.  eps is of the order of the clipped gradients, so the trajectory
    depends on coef (Adam alone is nearly scale-invariant); some steps are unclipped (norm below
    max_norm).  A coefficient computed on unscaled grads, per tensor instead of globally, applied
    before the scale or skipped would leave the tolerance."""
    import torch
    sizes, T, gs = [1000, 37, 2048], 12, 1.0 / 1024.0
    lr, b1, b2, eps, wd, max_norm = 1e-3, 0.9, 0.95, 1e-3, 0.1, 0.05
    ws = [synth.weights(n, 0.02, 0xB0B + i) for i, n in enumerate(sizes)]
    ps = [torch.nn.Parameter(torch.from_numpy(w.copy())) for w in ws]
    cls = torch.optim.AdamW if adamw else torch.optim.Adam
    opt = cls(ps, lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd, foreach=False, fused=False)
    ms = [np.zeros(n, np.float32) for n in sizes]
    vs = [np.zeros(n, np.float32) for n in sizes]
    wmax = [np.abs(w).astype(np.float64) for w in ws]
    clipped = 0
    for t in range(1, T + 1):
        sig = (2e-3 if t % 3 else 2e-4) * 1024.0      # every third step: norm < max_norm, coef = 1
        g16 = [synth.grads(n, sig, "fp16", 2023, 100 * t + i) for i, n in enumerate(sizes)]
        for p, g in zip(ps, g16):   # torch: unscale (fp32), then clip over all tensors, then step
            p.grad = torch.from_numpy(orc.widen("fp16", g) * np.float32(gs))
        torch.nn.utils.clip_grad_norm_(ps, max_norm, foreach=False)
        opt.step()
        S = sum(orc.sumsq("fp16", g, grad_scale=gs) for g in g16)
        coef = orc.clip_coef(S, max_norm)
        clipped += coef < 1.0
        for i in range(len(sizes)):
            orc.adam_step_master("fp16", ws[i], g16[i], ms[i], vs[i], lr=lr, beta1=b1, beta2=b2, eps=eps,
                                 weight_decay=wd, adamw=adamw, grad_scale=gs, step=t, clip_coef=coef)
            wmax[i] = np.maximum(wmax[i], np.abs(ws[i]))
    assert 0 < clipped < T
    for i in range(len(sizes)):
        ref = ps[i].detach().numpy().astype(np.float64)
        err = np.abs(ws[i].astype(np.float64) - ref)
        assert (err <= 2 * T * _ulp32(wmax[i])).all(), err.max()
    # the same run with the coefficient left out is far outside that tolerance (the test bites)
    w_noclip = ws[0].copy() * 0 + synth.weights(sizes[0], 0.02, 0xB0B)
    m0 = np.zeros(sizes[0], np.float32); v0 = np.zeros(sizes[0], np.float32)
    for t in range(1, T + 1):
        sig = (2e-3 if t % 3 else 2e-4) * 1024.0
        g = synth.grads(sizes[0], sig, "fp16", 2023, 100 * t)
        orc.adam_step_master("fp16", w_noclip, g, m0, v0, lr=lr, beta1=b1, beta2=b2, eps=eps, weight_decay=wd,
                             adamw=adamw, grad_scale=gs, step=t)
    ref = ps[0].detach().numpy().astype(np.float64)
    assert np.abs(w_noclip.astype(np.float64) - ref).max() > 100 * 2 * T * _ulp32(wmax[0]).max()


def test_adam_lerp_closed_forms(orc):
    """The first-moment update m <- lerp(m, g, 1-beta1) (R6) against its closed forms, both
    branches: beta1 = 0 gives m_new = g EXACTLY (the upper formula g - (g-m)*0; the lower one,
    m + 1*(g-m), would round g-m); beta1 = 0.5 on dyadic inputs is exact (m+g)/2; and for random
    inputs and beta1 in {0.9, 0.64, 0.5, 0.3, 0.1} m_new lies within 2 binary32 ulps (of the
    operands' scale) of the exact lerp computed in fp64.  Observed through Adam's m output on an fp32 master."""
    n = 1 << 14
    m0 = synth.normal_f32(n, 1e-2, 9, 1)
    g = synth.normal_f32(n, 1e-2, 9, 2)
    w = np.zeros(n, np.float32)
    m = m0.copy(); v = np.zeros(n, np.float32)
    orc.adam_step_master("fp32", w, g, m, v, lr=1e-3, beta1=0.0, step=2)
    assert np.array_equal(m.view(np.uint32), g.view(np.uint32))
    # the lower formula would not be exact here (the test distinguishes the branches)
    low = (m0 + (g - m0)).astype(np.float32)
    assert np.count_nonzero(low != g) > n // 4
    md = (np.round(m0 * 2 ** 12) / 2 ** 12).astype(np.float32)
    gd = (np.round(g * 2 ** 12) / 2 ** 12).astype(np.float32)
    m = md.copy(); v = np.zeros(n, np.float32)
    orc.adam_step_master("fp32", w.copy(), gd, m, v, lr=1e-3, beta1=0.5, step=2)
    assert np.array_equal(m, ((md.astype(np.float64) + gd.astype(np.float64)) / 2).astype(np.float32))
    for b1 in (0.9, 0.64, 0.5, 0.3, 0.1):
        wgt = np.float64(np.float32(1.0 - b1))          # the float lerp weight both sides use (R7)
        m = m0.copy(); v = np.zeros(n, np.float32)
        orc.adam_step_master("fp32", w.copy(), g, m, v, lr=1e-3, beta1=b1, step=2)
        exact = m0.astype(np.float64) + wgt * (g.astype(np.float64) - m0.astype(np.float64))
        # three roundings (g - m, the product, the sum): within 2 ulps of the operands' scale
        scale = np.maximum(np.abs(m0), np.abs(g))
        assert (np.abs(m.astype(np.float64) - exact) <= 2 * _ulp32(scale)).all(), b1
        # a branch with the weight's complement (the classic slip) is far outside
        wrong = m0.astype(np.float64) + (1 - wgt) * (g.astype(np.float64) - m0.astype(np.float64))
        assert np.median(np.abs(wrong - exact) / _ulp32(scale)) > 1000 or b1 == 0.5


# ----------------------------------------------------------------------------------- P9 --
def test_p9_byte_model(orc):
    # fp32 value + 16-bit copy = 6 B, grad "usually 4 bytes"; P:15 Adam state 8 B
    assert orc.bytes_per_param("amp", "adam") == 18
    assert orc.bytes_per_param("amp", "sgd_momentum") == 14
    # "at least 6 bytes less" with the residual and the fused backward
    assert orc.bytes_per_param("amp", "adam") - orc.bytes_per_param("ours_fused_backward", "adam") >= 6
    assert orc.bytes_per_param("ours_fused_backward", "adam") == 12
    assert orc.bytes_per_param("ours_fused_backward", "sgd_momentum") == 8
    assert orc.bytes_per_param("ours_multi_tensor", "adam") == 14


# ------------------------------------------------------------- clip-by-value ingest --
def test_clip_value_closed_form_and_torch_clamp(orc):
    """SPEC S:322 example: clip c=0.5, grad [1, -2, 0.1] -> effective grad [0.5, -0.5, 0.1]; and on
    random grads (with +-Inf, NaN) the oracle's ingest equals torch.clamp (library routine), seen
    through an SGD step with lr=1 from w=0 (w_new = -g_effective exactly)."""
    import torch
    g = np.array([1.0, -2.0, 0.1], np.float32)
    w = np.zeros(3, np.float32)
    orc.sgd_step_master("fp32", w, g, None, lr=1.0, clip_value=0.5)
    assert np.array_equal(-w, np.array([0.5, -0.5, np.float32(0.1)], np.float32))
    g = np.concatenate([synth.normal_f32(5000, 2.0, 3, 3), np.array([np.inf, -np.inf, np.nan, 0.0, -0.0], np.float32)])
    for c, gs in ((0.7, 1.0), (1.5, 0.25), (3.0, 2.0)):
        w = np.zeros(g.size, np.float32)
        orc.sgd_step_master("fp32", w, g, None, lr=1.0, grad_scale=gs, clip_value=c)
        want = torch.clamp(torch.from_numpy(g) * np.float32(gs), -np.float32(c), np.float32(c)).numpy()
        got = -w
        nan = np.isnan(want)
        assert np.array_equal(np.isnan(got), nan) and np.array_equal(got[~nan], want[~nan])
    # clip_value 0 = off: identical to the unclipped step
    w1 = np.zeros(g.size, np.float32); w2 = np.zeros(g.size, np.float32)
    orc.sgd_step_master("fp32", w1, g, None, lr=1.0, clip_value=0.0)
    orc.sgd_step_master("fp32", w2, g, None, lr=1.0)
    assert np.array_equal(w1.view(np.uint32), w2.view(np.uint32))


def test_clip_value_in_residual_steps_matches_master(orc):
    """The residual-compensated Adam / SGD steps apply the same ingest (bf16: value+residual equal
    the clipped fp32-master trajectory on every element without a lossy split)."""
    n = 4096
    w = synth.weights(n, 0.02, 11)
    g = synth.grads(n, 5e-2, "bf16", 11, 1)
    for kind in ("adam", "sgd"):
        h, r = orc.split("bf16", w)
        wm = w.copy()
        m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
        mm = np.zeros(n, np.float32); vm = np.zeros(n, np.float32)
        if kind == "adam":
            orc.adam_step("bf16", "bf16", h, r, g, m, v, lr=1e-3, clip_value=0.03)
            orc.adam_step_master("bf16", wm, g, mm, vm, lr=1e-3, clip_value=0.03)
        else:
            orc.sgd_step("bf16", "bf16", h, r, g, m, lr=0.1, momentum=0.9, first_step=True, clip_value=0.03)
            orc.sgd_step_master("bf16", wm, g, mm, lr=0.1, momentum=0.9, first_step=True, clip_value=0.03)
        rec = orc.reconstruct("bf16", h, r)
        lossy = (r == 32767)
        assert np.array_equal(rec.view(np.uint32)[~lossy], wm.view(np.uint32)[~lossy])
        assert np.array_equal(m, mm)


# ------------------------------------------------------------------------------------------
# R15: reduction over ranks of the P2P fused sharded step (BJ north_star (c))
# ------------------------------------------------------------------------------------------
def test_reduce_sum16_world1_is_the_exact_widening(orc):
    """One rank: the 'sum' is the gradient widened to binary32, i.e. numpy's own exact
    float16 -> float32 cast (library routine), over all 2^16 fp16 patterns."""
    h = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    out = orc.reduce_sum16("fp16", [h])
    ref = h.view(np.float16).astype(np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(out), nan)
    assert np.array_equal(out[~nan].view(np.uint32), ref[~nan].view(np.uint32))


def test_reduce_sum16_exact_when_no_rounding_and_bound_otherwise(orc):
    """Exact-sum construction: multiples of 2^-10 below 2^10 summed over 8 ranks are exact in
    binary32, so the result equals math.fsum of the widened values.  Random gradients: the error
    of recursive summation obeys |s - exact| <= (W-1) u sum|g_k| (u = 2^-24, Higham)."""
    import math
    rng = np.random.default_rng(2023)
    W, n = 8, 4096
    ks = [rng.integers(-2 ** 20, 2 ** 20, n) for _ in range(W)]
    gs = [(k.astype(np.float64) * 2.0 ** -10).astype(np.float16).view(np.uint16) for k in ks]
    exact = np.array([math.fsum(float(g.view(np.float16)[i]) for g in gs) for i in range(n)])
    out = orc.reduce_sum16("fp16", gs)
    assert np.array_equal(out.astype(np.float64), exact)
    gs = [rng.normal(0, 1, n).astype(np.float16).view(np.uint16) for _ in range(W)]
    wid = [g.view(np.float16).astype(np.float64) for g in gs]
    exact = np.array([math.fsum(w[i] for w in wid) for i in range(n)])
    bound = (W - 1) * 2.0 ** -24 * np.sum(np.abs(np.stack(wid)), axis=0)
    out = orc.reduce_sum16("fp16", gs).astype(np.float64)
    assert np.all(np.abs(out - exact) <= bound)
    assert np.any(out != exact)          # rounding really happens: the test is not vacuous


def test_reduce_sum16_is_in_rank_order(orc):
    """bf16: 2^24 + 1 + 1 in binary32 is 2^24 in rank order ((2^24 + 1) ties to even), but
    2^24 + 2 if the two ones were added first: the oracle adds in rank order."""
    big, one = np.array([0x4B80], np.uint16), np.array([0x3F80], np.uint16)   # 2^24, 1.0 in bf16
    assert orc.reduce_sum16("bf16", [big, one, one])[0] == np.float32(2.0 ** 24)
    assert orc.reduce_sum16("bf16", [one, one, big])[0] == np.float32(2.0 ** 24 + 2)
