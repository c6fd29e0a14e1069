"""GPU parity at the edges of the number formats: whole optimizer steps, bit-exact (exact build)
against the oracle, on UNSCALED edge weights and non-finite / extreme gradients.

Weights: synth.edge_f32() as they are (+-0, fp32 subnormals, RNE ties, 65504 / just below 65520 /
65520, the bf16 max-finite boundary 0x7F7F8000.., 2^-17 .. 2^-24, +-Inf, NaN), plus the largest
finite fp16 / bf16 values and their negatives, so an update can overflow a value to +-Inf or
start at the largest finite one.  Gradients: +-0, the smallest and largest subnormals, the
largest finite value of the gradient's format (fp16 65504, bf16 0x7F7F, fp32 FLT_MAX), +-Inf,
NaN, 1.0 and ordinary small values.  Every weight meets every gradient (their cross product laid
out in 8-element units and in ragged tails), through every storage format, SGD-momentum /
Nesterov and Adam / AdamW / Adam-L2, two consecutive steps (m, v carried), fp32 and 16-bit
gradients.  Value, residual, m and v are compared element by element (m/v: any NaN equals any
NaN, R8).  Reference: P:70 (reconstruct -> update -> re-split), P:82 (Adam, SGD),
P:84 (rounding), readings R3-R5 (ties, NaN/Inf, subnormals), R14 (variants).
"""
import numpy as np
import pytest
import torch

from gpu_util import TDT, dev16, dev_grad, devf, host16, same_bits_nan_equal
import synth

pytestmark = pytest.mark.gpu

FORMATS = [("rne", "fp16"), ("rne", "bf16"), ("rtz", "fp16"), ("rtz", "bf16"), ("sr", "fp16"), ("x8", "fp16"),
           ("x8", "bf16"), ("x8z", "fp16"), ("x8z", "bf16")]
RDT = {"rne": np.int16, "rtz": np.uint16, "sr": np.int16, "x8": np.int8, "x8z": np.uint8}

EDGE_G = {
    # +-0, min / max subnormal, max finite (both signs), +-Inf, NaN, 1.0, a normal small value
    "fp16": [0x0000, 0x8000, 0x0001, 0x83FF, 0x7BFF, 0xFBFF, 0x7C00, 0xFC00, 0x7E00, 0x3C00, 0x1E00, 0x9400],
    "bf16": [0x0000, 0x8000, 0x0001, 0x807F, 0x7F7F, 0xFF7F, 0x7F80, 0xFF80, 0x7FC0, 0x3F80, 0x3A80, 0xBC00],
    "fp32": [0x00000000, 0x80000000, 0x00000001, 0x807FFFFF, 0x7F7FFFFF, 0xFF7FFFFF, 0x7F800000, 0xFF800000,
             0x7FC00000, 0x3F800000, 0x3A800000, 0xBC000000],
}


@pytest.fixture(scope="module")
def mpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_12381_b200 as m
    from paper_2309_12381_b200 import _build
    _build.build()
    return m


def edge_weights(fmt):
    extra = np.array([0x477FE000, 0xC77FE000, 0x7F7F0000, 0xFF7F0000, 0x3C23D70A, 0xBC23D70A],
                     np.uint32).view(np.float32)   # fp16 / bf16 largest finite, +-0.01
    return np.concatenate([synth.edge_f32(), extra]).astype(np.float32)


def cross(fmt, gfmt, shift):
    """Every edge weight with every edge gradient; `shift` rotates the pairing so a combination
    lands both inside full 8-element units and in ragged tails across the tensors."""
    w = edge_weights(fmt)
    g = np.array(EDGE_G[gfmt], np.uint32 if gfmt == "fp32" else np.uint16)
    nw, ng = w.size, g.size
    i = np.arange(nw * ng)
    W = w[(i + shift) % nw]
    G = g[(i // nw + shift) % ng]
    if gfmt == "fp32":
        G = G.view(np.float32)
    return W, np.ascontiguousarray(G)


def state(n, seed):
    m = synth.normal_f32(n, 1e-3, seed, 1)
    v = np.abs(synth.normal_f32(n, 1e-5, seed, 2))
    # a few extreme optimizer states: 0, subnormal, huge, +-Inf / NaN moments
    sp = np.array([0.0, 1e-45, 3e38, np.inf, np.nan, -np.inf], np.float32)
    m[::37] = sp[np.arange(m[::37].size) % sp.size]
    v[::41] = np.abs(sp[np.arange(v[::41].size) % sp.size])
    return m, v


def dev_resid(r):
    if r.dtype in (np.int8, np.uint8):
        return torch.from_numpy(r.copy()).cuda()
    return torch.from_numpy(np.ascontiguousarray(r).view(np.int16).copy()).cuda()


def host_resid(t, scheme):
    a = t.cpu().numpy()
    return a.view(RDT[scheme]) if scheme not in ("x8", "x8z") else a


KINDS = ["adamw", "adam_l2", "adam_b1_0", "sgd_m", "sgd_nesterov"]


def _hps(mpo, kind, t, seed):
    if kind == "adamw":
        return mpo.AdamParams(lr=1e-3, beta1=0.9, beta2=0.999, weight_decay=0.1, adamw=True, step=t, seed=seed)
    if kind == "adam_l2":
        return mpo.AdamParams(lr=2e-2, beta1=0.9, beta2=0.95, weight_decay=0.01, adamw=False, step=t,
                              grad_scale=0.5, seed=seed)
    if kind == "adam_b1_0":
        return mpo.AdamParams(lr=5e-4, beta1=0.0, beta2=0.9, eps=1e-6, step=t, seed=seed)
    if kind == "sgd_m":
        return mpo.SgdParams(lr=0.3, momentum=0.9, weight_decay=2e-4, first_step=(t == 1), seed=seed)
    return mpo.SgdParams(lr=0.5, momentum=0.9, nesterov=True, first_step=(t == 1), grad_scale=2.0, seed=seed)


@pytest.mark.parametrize("scheme,fmt", FORMATS)
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gsame", [True, False])
def test_edge_steps_bit_exact(mpo, orc, scheme, fmt, kind, gsame, step_kernel):
    gf = fmt if gsame else "fp32"
    hs, rs, gs, ms, vs = [], [], [], [], []
    for shift in range(3):
        W, G = cross(fmt, gf, shift)
        if shift == 2:                      # a ragged tensor: tail of 5 (X8: 16-element granule)
            W, G = W[:-5], G[:-5]
        h, r = orc.split_s(scheme, fmt, W, seed=5, stream=shift)
        m, v = state(W.size, 40 + shift)
        hs.append(h); rs.append(r); gs.append(G); ms.append(m); vs.append(v)
    # sanity: the weights really are unscaled (65504, bf16 max-finite and Inf are present)
    assert np.isin(np.array([0x7BFF, 0x7C00] if fmt == "fp16" else [0x7F7F, 0x7F80], np.uint16), hs[0]).all()
    V = [dev16(h, fmt) for h in hs]
    R = [dev_resid(r) for r in rs]
    M = [devf(m) for m in ms]
    Wv = [devf(v) for v in vs]
    adam = kind.startswith("adam")
    for t in (1, 2):
        seed = 900 + t
        hp = _hps(mpo, kind, t, seed)
        G = [dev_grad(g, gf) for g in gs]
        tab = mpo.TensorTable(V, R, G, M, Wv if adam else [None] * len(V), scheme=scheme)
        if adam:
            mpo.mpo_adam_step(tab, hp, exact=True)
        else:
            mpo.mpo_sgd_step(tab, hp, exact=True)
        for i in range(len(V)):
            g_in = gs[i]
            if adam:
                orc.adam_step_s(scheme, fmt, gf, hs[i], rs[i], g_in, ms[i], vs[i], seed=seed, stream=i,
                                lr=hp.lr, beta1=hp.beta1, beta2=hp.beta2, eps=hp.eps, weight_decay=hp.weight_decay,
                                adamw=hp.adamw, grad_scale=hp.grad_scale, step=hp.step)
            else:
                orc.sgd_step_s(scheme, fmt, gf, hs[i], rs[i], g_in, ms[i], lr=hp.lr, momentum=hp.momentum,
                               weight_decay=hp.weight_decay, nesterov=hp.nesterov, first_step=hp.first_step,
                               grad_scale=hp.grad_scale, seed=seed, stream=i)
        for i in range(len(V)):
            hg = host16(V[i])
            bad = np.flatnonzero(hg != hs[i])
            assert bad.size == 0, (t, i, bad[:5], hg[bad[:5]], hs[i][bad[:5]])
            assert np.array_equal(host_resid(R[i], scheme), rs[i]), (t, i)
            assert same_bits_nan_equal(M[i].cpu().numpy(), ms[i]), (t, i)
            if adam:
                assert same_bits_nan_equal(Wv[i].cpu().numpy(), vs[i]), (t, i)
    # the cases the test claims are really reached: finite weights that overflowed to +-Inf or
    # became NaN in these two steps, and finite results from the largest finite weights
    inf16 = np.array((0x7C00, 0xFC00) if fmt == "fp16" else (0x7F80, 0xFF80), np.uint16)
    nonfin = lambda h: np.isin(h, inf16) | (h == 0x7FFF)
    h0 = np.concatenate([orc.split_s(scheme, fmt, cross(fmt, gf, k)[0][:len(hs[k])], seed=5, stream=k)[0]
                         for k in range(3)])
    h_all = np.concatenate(hs)
    assert (~nonfin(h0) & nonfin(h_all)).any()
    maxf = np.array((0x7BFF, 0xFBFF) if fmt == "fp16" else (0x7F7F, 0xFF7F), np.uint16)
    assert (np.isin(h0, maxf) & ~nonfin(h_all)).any() or kind in ("adam_l2", "sgd_m")


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("kind", ["adamw", "sgd_m"])
def test_edge_hook_step_bit_exact(mpo, orc, fmt, kind):
    """The hook entry point (one tensor) on the same edge cross product, ragged length."""
    from paper_2309_12381_b200._lib import MPO_ADAM, MPO_SGD, Tensor
    from paper_2309_12381_b200 import api
    W, G = cross(fmt, fmt, 1)
    W, G = W[:-3], G[:-3]
    h, r = orc.split(fmt, W)
    m, v = state(W.size, 77)
    V, R, Gd, M, Vv = dev16(h, fmt), dev_resid(r), dev_grad(G, fmt), devf(m), devf(v)
    row = Tensor()
    row.value, row.resid, row.grad, row.m, row.v = V.data_ptr(), R.data_ptr(), Gd.data_ptr(), M.data_ptr(), Vv.data_ptr()
    row.n = W.size
    hp = _hps(mpo, kind, 1, 0)
    api.mpo_fused_backward_hook_step(MPO_ADAM if kind == "adamw" else MPO_SGD, api.format_code(TDT[fmt]),
                                     api.dtype_code(TDT[fmt]), row, hp.c(), exact=True)
    if kind == "adamw":
        orc.adam_step(fmt, fmt, h, r, G, m, v, lr=hp.lr, beta1=hp.beta1, beta2=hp.beta2, eps=hp.eps,
                      weight_decay=hp.weight_decay, adamw=hp.adamw, step=1)
    else:
        orc.sgd_step(fmt, fmt, h, r, G, m, lr=hp.lr, momentum=hp.momentum, weight_decay=hp.weight_decay,
                     first_step=True)
    assert np.array_equal(host16(V), h)
    assert np.array_equal(R.cpu().numpy(), r)
    assert same_bits_nan_equal(M.cpu().numpy(), m)
    if kind == "adamw":
        assert same_bits_nan_equal(Vv.cpu().numpy(), v)


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("kind", ["adamw", "sgd_m"])
def test_edge_steps_fma_build(mpo, orc, fmt, kind):
    """The FMA build (exact=False) on the same edge cross product: every special outcome is the
    oracle's exactly (NaN -> 0x7FFF, +-Inf, signed zeros, overflow to Inf at the same elements), and
    the finite values are within 1 ulp16 or R12's operand-scaled bound of the oracle."""
    from gpu_util import ulp16_dist
    W, G = cross(fmt, fmt, 0)
    h, r = orc.split(fmt, W)
    m, v = state(W.size, 91)
    V, R, Gd, M, Vv = dev16(h, fmt), dev_resid(r), dev_grad(G, fmt), devf(m), devf(v)
    hp = _hps(mpo, kind, 2, 0)
    adam = kind == "adamw"
    tab = mpo.TensorTable([V], [R], [Gd], [M], [Vv] if adam else [None])
    if adam:
        mpo.mpo_adam_step(tab, hp, exact=False)
        orc.adam_step(fmt, fmt, h, r, G, m, v, lr=hp.lr, beta1=hp.beta1, beta2=hp.beta2, eps=hp.eps,
                      weight_decay=hp.weight_decay, adamw=hp.adamw, step=hp.step)
    else:
        mpo.mpo_sgd_step(tab, hp, exact=False)
        orc.sgd_step(fmt, fmt, h, r, G, m, lr=hp.lr, momentum=hp.momentum, weight_decay=hp.weight_decay,
                     first_step=hp.first_step)
    hg = host16(V)
    inf16 = (0x7C00, 0xFC00) if fmt == "fp16" else (0x7F80, 0xFF80)
    special = lambda x: np.isin(x, np.array(inf16 + (0x7FFF,), np.uint16))
    assert np.array_equal(special(hg), special(h))
    assert np.array_equal(hg[special(h)], h[special(h)])
    fin = ~special(h)
    wg = orc.reconstruct(fmt, hg, R.cpu().numpy().view(np.int16)).astype(np.float64)
    wo = orc.reconstruct(fmt, h, r).astype(np.float64)
    w0 = W.astype(np.float64)
    close = (ulp16_dist(hg, h, fmt) <= 1) | (np.abs(wg - wo) <= 1e-6 * (np.abs(w0) + np.abs(wo)) + 2.0 ** -24)
    assert close[fin].all(), np.flatnonzero(fin & ~close)[:8]
