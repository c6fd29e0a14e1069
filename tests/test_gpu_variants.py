"""GPU parity of the paper variants of the storage scheme against the CPU oracle.

* split / reconstruct under RTZ (fp16, bf16), SR (fp16), X8 and X8Z (fp16, bf16): bit-exact on ALL 2^32
  binary32 patterns (SR with the shared counter-based draws keyed by (seed, stream, index));
* Adam / AdamW / SGD-momentum steps through the multi-tensor table, ragged sizes (tails of X8's
  16-element bulk-copy granule included), several hyper-parameter groups and streams: bit-exact
  in the -fmad=false build, every step;
* the optimizer objects: hook mode == multi-tensor mode bitwise under SR (per-parameter streams).
"""
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import synth
from gpu_util import TDT, bits32, dev16, dev_grad, devf, hostf, host16, same_bits_nan_equal

pytestmark = pytest.mark.gpu

VARIANTS = [("rtz", "fp16"), ("rtz", "bf16"), ("sr", "fp16"), ("x8", "fp16"), ("x8", "bf16"), ("x8z", "fp16"),
            ("x8z", "bf16")]
RDT = {"rne": np.int16, "rtz": np.uint16, "sr": np.int16, "x8": np.int8, "x8z": np.uint8}


@pytest.fixture(scope="module")
def mpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_12381_b200 as m
    from paper_2309_12381_b200 import _build
    _build.build()
    return m


def dev_resid(r):
    if r.dtype in (np.int8, np.uint8):
        return torch.from_numpy(r.copy()).cuda()
    return torch.from_numpy(np.ascontiguousarray(r).view(np.int16).copy()).cuda()


def host_resid(t, scheme):
    a = t.cpu().numpy()
    return a.view(RDT[scheme]) if scheme not in ("x8", "x8z") else a


@pytest.mark.parametrize("scheme,fmt", VARIANTS)
def test_variant_split_reconstruct_all_2_32(mpo, orc, scheme, fmt):
    chunk = 1 << 26
    lock = threading.Lock()
    seed = 0xC0FFEE

    def one(c):
        u = np.arange(c * chunk, (c + 1) * chunk, dtype=np.uint64).astype(np.uint32)
        x = u.view(np.float32)
        ho, ro = orc.split_s(scheme, fmt, x, seed=seed + c, stream=3)
        reco = orc.reconstruct_s(scheme, fmt, ho, ro)
        with lock:
            v, r = mpo.mpo_split(devf(x), TDT[fmt], scheme=scheme, seed=seed + c, sr_stream=3)
            rec = mpo.mpo_reconstruct(v, r, scheme=scheme)
            hg, rg, recg = host16(v), host_resid(r, scheme), hostf(rec)
        return int(np.count_nonzero(hg != ho)) + int(np.count_nonzero(rg != ro)) + \
            int(np.count_nonzero(bits32(recg) != bits32(reco)))

    with ThreadPoolExecutor(max_workers=max(2, min(16, os.cpu_count() or 2))) as ex:
        assert sum(ex.map(one, range(64))) == 0


SIZES = [0, 1, 7, 8, 9, 15, 16, 17, 4095, 4096, 4097, 12345, 65539, 3]


def _kw(hp):
    return dict(lr=hp.lr, beta1=hp.beta1, beta2=hp.beta2, eps=hp.eps, weight_decay=hp.weight_decay,
                adamw=hp.adamw, grad_scale=hp.grad_scale, step=hp.step)


@pytest.mark.parametrize("scheme,fmt", VARIANTS)
@pytest.mark.parametrize("kind", ["adam", "sgd"])
@pytest.mark.parametrize("gsame", [True, False])
def test_variant_steps_bit_exact(mpo, orc, scheme, fmt, kind, gsame, step_kernel):
    gf = fmt if gsame else "fp32"
    hs, rs, ms, vs = [], [], [], []
    for i, n in enumerate(SIZES):
        w = synth.weights(n, 0.05, 0xB0B + i)
        if n > 40:
            w[:36] = synth.edge_f32() * np.float32(1e-3)
        if n > 80:
            w[36:72] = synth.edge_f32()      # unscaled: overflow, Inf, NaN, max-finite
        h, r = orc.split_s(scheme, fmt, w, seed=77, stream=i)
        hs.append(h); rs.append(r)
        ms.append(synth.normal_f32(n, 1e-3, 5, i)); vs.append(np.abs(synth.normal_f32(n, 1e-5, 6, i)))
    V = [dev16(h, fmt) for h in hs]
    R = [dev_resid(r) for r in rs]
    M = [devf(m) for m in ms]
    W = [devf(v) for v in vs]
    grp = [i % 2 for i in range(len(SIZES))]
    for t in range(1, 4):
        gs = [synth.grads(n, 1e-2, gf, 0xC0FFEE + t, i) for i, n in enumerate(SIZES)]
        G = [dev_grad(g, gf) for g in gs]
        seed = 1000 + t
        if kind == "adam":
            hps = [mpo.AdamParams(lr=1e-3, weight_decay=0.1, adamw=True, step=t, seed=seed),
                   mpo.AdamParams(lr=2e-3, beta2=0.95, weight_decay=0.01, adamw=False, step=t, grad_scale=0.5,
                                  seed=seed)]
            tab = mpo.TensorTable(V, R, G, M, W, grp, scheme=scheme)
            mpo.mpo_adam_step(tab, hps, exact=True)
        else:
            hps = [mpo.SgdParams(lr=0.1, momentum=0.9, weight_decay=1e-4, first_step=(t == 1), seed=seed),
                   mpo.SgdParams(lr=0.05, momentum=0.9, nesterov=True, first_step=(t == 1), seed=seed)]
            tab = mpo.TensorTable(V, R, G, M, [None] * len(SIZES), grp, scheme=scheme)
            mpo.mpo_sgd_step(tab, hps, exact=True)
        for i, n in enumerate(SIZES):
            hp = hps[grp[i]]
            if kind == "adam":
                orc.adam_step_s(scheme, fmt, gf, hs[i], rs[i], gs[i], ms[i], vs[i], seed=seed, stream=i, **_kw(hp))
            else:
                orc.sgd_step_s(scheme, fmt, gf, hs[i], rs[i], gs[i], ms[i], lr=hp.lr, momentum=hp.momentum,
                               weight_decay=hp.weight_decay, nesterov=hp.nesterov, first_step=hp.first_step,
                               seed=seed, stream=i)
    for i in range(len(SIZES)):
        assert np.array_equal(host16(V[i]), hs[i]), (i, SIZES[i])
        assert np.array_equal(host_resid(R[i], scheme), rs[i]), (i, SIZES[i])
        assert same_bits_nan_equal(M[i].cpu().numpy(), ms[i]), i
        if kind == "adam":
            assert same_bits_nan_equal(W[i].cpu().numpy(), vs[i]), i


@pytest.mark.parametrize("scheme,fmt,native", [("sr", torch.float16, True), ("sr", torch.float16, False),
                                               ("rtz", torch.bfloat16, True), ("x8", torch.float16, True),
                                               ("x8", torch.bfloat16, False), ("x8z", torch.float16, True),
                                               ("x8z", torch.bfloat16, False)])
def test_variant_hook_mode_equals_multi_tensor(mpo, scheme, fmt, native):
    """Every storage variant through the fused backward (native C++ and Python hooks): == the
    multi-tensor step bitwise; stochastic rounding is keyed by per-parameter streams, so both paths
    draw the same numbers."""
    torch.manual_seed(0)
    d = 96
    mk = lambda: torch.nn.Sequential(torch.nn.Linear(d, 2 * d), torch.nn.GELU(), torch.nn.Linear(2 * d, d)).cuda()
    a, b = mk(), mk()
    b.load_state_dict(a.state_dict())
    oa = mpo.ResidualAdamW(a.parameters(), lr=1e-3, weight_decay=0.1, fmt=fmt, scheme=scheme, seed=9)
    ob = mpo.ResidualAdamW(b.parameters(), lr=1e-3, weight_decay=0.1, fmt=fmt, scheme=scheme, seed=9)
    ob.install_backward_hooks(native=native, batch_below=0 if native else 1 << 16)
    for t in range(3):
        x = torch.randn(32, d, device="cuda", dtype=fmt)
        a(x).float().square().mean().backward()
        oa.step()
        for p in a.parameters():
            p.grad = None
        b(x).float().square().mean().backward()
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert torch.equal(pa.view(torch.int16), pb.view(torch.int16))
        assert torch.equal(oa.state[pa]["resid"], ob.state[pb]["resid"])


@pytest.mark.parametrize("scheme,fmt,kind", [("rne", "bf16", "adam"), ("x8", "fp16", "sgd"), ("rne", "fp16", "sgd")])
def test_schedule_many_tensors_with_guards(mpo, orc, scheme, fmt, kind, step_kernel):
    """The step kernel's schedule (tiles dealt round-robin to the CTAs, each
    stage's piece published by the producer warp): 400 tensors of mixed sizes (empty, tiny,
    ragged, several tiles) over every CTA, more tiles than one wave, tails of the int8 residual's
    16-element granule.  Every tensor is a view into a flat buffer with a guard gap after it: the
    exact build matches the oracle bit for bit and no guard word changes."""
    rng = np.random.default_rng(2023)
    sizes = [int(s) for s in rng.choice([0, 1, 3, 8, 15, 16, 17, 64, 100, 4095, 4096, 4097, 9000, 20011], 400)]
    GUARD = 64   # elements after every tensor (keeps every view 16-B aligned for any residual width)
    offs, o = [], 0
    for n in sizes:
        offs.append(o)
        o += (n + 15) // 16 * 16 + GUARD
    total = o
    rdt = RDT[scheme]
    hs, rs, ms, vs, gs = [], [], [], [], []
    for i, n in enumerate(sizes):
        w = synth.weights(n, 0.05, 0xB0B + i)
        h, r = orc.split_s(scheme, fmt, w, seed=5, stream=i)
        hs.append(h); rs.append(r)
        ms.append(synth.normal_f32(n, 1e-3, 5, i)); vs.append(np.abs(synth.normal_f32(n, 1e-5, 6, i)))
        gs.append(synth.grads(n, 1e-2, fmt, 0xC0FFEE, i))
    # flat host images, guards filled with a recognisable pattern
    fh = np.full(total, 0x7E57, np.uint16)
    fr = np.full(total, 0x55 if rdt == np.int8 else 0x5A5A, np.uint8 if rdt == np.int8 else np.uint16)
    fg = np.full(total, 0x3C00, np.uint16)
    fm = np.full(total, 7.0, np.float32)
    fv = np.full(total, 9.0, np.float32)
    for i, n in enumerate(sizes):
        s = slice(offs[i], offs[i] + n)
        fh[s] = hs[i]; fr[s] = rs[i].view(fr.dtype); fg[s] = gs[i]; fm[s] = ms[i]; fv[s] = vs[i]
    H, G = dev16(fh, fmt), dev16(fg, fmt)
    R = torch.from_numpy(fr.view(np.int8 if rdt == np.int8 else np.int16).copy()).cuda()
    M, W = devf(fm), devf(fv)
    view = lambda t, i: t[offs[i]:offs[i] + sizes[i]]
    grp = [i % 2 for i in range(len(sizes))]
    if kind == "adam":
        hps = [mpo.AdamParams(lr=1e-3, weight_decay=0.1, adamw=True, step=2),
               mpo.AdamParams(lr=2e-3, beta2=0.95, step=2, grad_scale=0.5)]
        tab = mpo.TensorTable([view(H, i) for i in range(len(sizes))], [view(R, i) for i in range(len(sizes))],
                              [view(G, i) for i in range(len(sizes))], [view(M, i) for i in range(len(sizes))],
                              [view(W, i) for i in range(len(sizes))], grp, scheme=scheme)
        mpo.mpo_adam_step(tab, hps, exact=True)
    else:
        hps = [mpo.SgdParams(lr=0.1, momentum=0.9, weight_decay=1e-4),
               mpo.SgdParams(lr=0.05, momentum=0.9, nesterov=True)]
        tab = mpo.TensorTable([view(H, i) for i in range(len(sizes))], [view(R, i) for i in range(len(sizes))],
                              [view(G, i) for i in range(len(sizes))], [view(M, i) for i in range(len(sizes))],
                              [None] * len(sizes), grp, scheme=scheme)
        mpo.mpo_sgd_step(tab, hps, exact=True)
    for i, n in enumerate(sizes):
        hp = hps[grp[i]]
        if kind == "adam":
            orc.adam_step_s(scheme, fmt, fmt, hs[i], rs[i], gs[i], ms[i], vs[i], seed=0, stream=i, **_kw(hp))
        else:
            orc.sgd_step_s(scheme, fmt, fmt, hs[i], rs[i], gs[i], ms[i], lr=hp.lr, momentum=hp.momentum,
                           weight_decay=hp.weight_decay, nesterov=hp.nesterov, first_step=hp.first_step,
                           seed=0, stream=i)
        s = slice(offs[i], offs[i] + n)
        fh[s] = hs[i]; fr[s] = rs[i].view(fr.dtype); fm[s] = ms[i]
        if kind == "adam":
            fv[s] = vs[i]
    assert np.array_equal(host16(H), fh), "value (tensor or guard) differs"
    assert np.array_equal(R.cpu().numpy().view(fr.dtype), fr), "residual (tensor or guard) differs"
    assert np.array_equal(M.cpu().numpy().view(np.uint32), fm.view(np.uint32)), "m (tensor or guard) differs"
    assert np.array_equal(W.cpu().numpy().view(np.uint32), fv.view(np.uint32)), "v (tensor or guard) differs"
    assert np.array_equal(host16(G), fg), "gradients must be read-only"


def test_forward_error_of_in_place_addition(mpo):
    """Fig. rstoc through the GPU step (scripts/error_bench.py): K = 200 in-place
    additions of N(0,1) tensors (the SGD step with lr = -1).  With 13 / 16 extra bits every scheme
    (RNE, RTZ, SR) gives exactly fp32's result, element by element (those bits "maintain a
    full fp32 accuracy"); with 8 extra bits (X8) the forward error lies between fp32's and
    classical fp16's."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "error_bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts",
                                    "error_bench.py"))
    eb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(eb)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    n, K = 1 << 16, 200
    a = torch.randn(n, device="cuda", generator=gen)
    bs = [torch.randn(n, device="cuda", generator=gen).half() for _ in range(K)]
    ref = None
    for s in ("rne", "rtz", "sr"):
        got, exact = eb.accumulate(mpo, a, bs, s)
        v, r = mpo.mpo_split(a, torch.float16, scheme=s, seed=1234, sr_stream=0)
        acc = mpo.mpo_reconstruct(v, r, scheme=s)         # the stored start, then fp32 additions
        keep = acc.abs() >= 2.0 ** -16                    # lossless range of the fp16 residual (R5)
        for b in bs:
            acc = acc + b.float()
        assert torch.equal(got.float()[keep], acc[keep]), s
        ref = eb._metrics(got, exact)["rel_err"] if s == "rne" else ref
    e8 = {}
    for s in ("x8", "x8z"):
        got, exact = eb.accumulate(mpo, a, bs, s)
        e8[s] = eb._metrics(got, exact)["rel_err"]
    a16 = a.half()
    acc16 = a16.clone()
    for b in bs:
        acc16 += b
    e16 = eb._metrics(acc16.double(), a16.double() + sum(b.double() for b in bs))["rel_err"]
    assert ref < e8["x8"] < e16 and ref < e8["x8z"] < e16, (ref, e8, e16)
    assert e8["x8"] < e8["x8z"]        # truncated extra bits (the paper's fp16+8) drift faster than rounded ones
