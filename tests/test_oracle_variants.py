"""Pins of the oracle's paper variants of the storage scheme (no GPU).

* RTZ ("saving only the first part of the 32bit significand is equivalent to applying a
  round-to-zero"): exhaustive 2^32 property sweep of the defining inequality |widen(h)| <= |x| <
  |widen(next(h))|, an independent brute-force search over all fp16 magnitudes on samples, and
  the paper's claim that 16 extra bits keep bf16 at full fp32 accuracy: lossless on EVERY
  finite pattern; fp16 lossless on [2^-17, 2^16).
* SR (P:84 stochastic rounding + "un-round" bit): the value is one of the two neighbours, the
  extreme draws give the closed forms, the rounding is unbiased (statistical bound), the signed
  difference reconstructs exactly on the fp16 normal range; the shared counter-based generator is
  uniform.
* X8 ("keeping only part of those bits", P:134 fp16+8): the value is the RNE value, the
  reconstruction error is at most half the kept quantum except at saturation.
* X8Z, the paper's own fp16+8 / bf16+8 ("saving only the first part of the 32bit
  significand"): RTZ value + the next 8 significand bits truncated, i.e. split +
  reconstruct = the binary32 pattern with its low 5 (fp16) / 8 (bf16) bits cleared, on every
  pattern of a stratified sample of all exponents (each 16-bit high half x 64 low halves).
* Trajectories: bf16 RTZ Adam is BIT-IDENTICAL to the fp32-master trajectory on every element
  (lossless storage, an independent numpy/oracle master loop); fp16 SR equals it on every element
  that never went below 2^-15; X8 stays within its per-step bound.
"""
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import oracle
import synth


def _nan32(u):
    return (u & 0x7FFFFFFF) > 0x7F800000


def _mag(u):
    return (u & 0x7FFFFFFF).astype(np.int64)


def _rtz_chunk(args):
    fmt, lo, n = args
    oracle.lib()
    u = np.arange(lo, lo + n, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    h, r = oracle.split_s("rtz", fmt, x)
    wb = oracle.widen(fmt, h).view(np.uint32)
    nan = _nan32(u)
    inf = (u & 0x7FFFFFFF) == 0x7F800000
    fin = ~nan & ~inf
    bad = 0
    # sign preserved (or zero)
    bad += int(np.count_nonzero(fin & ((wb ^ u) & 0x80000000 != 0) & ((wb & 0x7FFFFFFF) != 0)))
    # |widen(h)| <= |x|
    bad += int(np.count_nonzero(fin & (_mag(wb) > _mag(u))))
    # next magnitude exceeds |x| unless h is the largest finite value
    hm = h & 0x7FFF
    maxfin = 0x7BFF if fmt == "fp16" else 0x7F7F
    nxt = ((h & 0x8000) | (hm + 1)).astype(np.uint16)
    wn = oracle.widen(fmt, nxt).view(np.uint32)
    bad += int(np.count_nonzero(fin & (hm != maxfin) & (_mag(wn) <= _mag(u))))
    rec = oracle.reconstruct_s("rtz", fmt, h, r).view(np.uint32)
    lossy = fin & (rec != u)
    if fmt == "bf16":
        lossy_bad = int(np.count_nonzero(lossy))
    else:
        a = u & 0x7FFFFFFF
        in_range = (a >= 0x37000000) & (a < 0x47800000)          # [2^-17, 2^16)
        lossy_bad = int(np.count_nonzero(lossy & in_range))
    nan_ok = bool((h[nan] == 0x7FFF).all() and not r[nan].any())
    return bad, lossy_bad, nan_ok, int(np.count_nonzero(lossy))


@pytest.fixture(scope="module")
def rtz_sweeps():
    chunk = 1 << 26
    out = {}
    with ProcessPoolExecutor(max_workers=max(2, min(8, os.cpu_count() or 2))) as ex:
        for fmt in ("bf16", "fp16"):
            out[fmt] = list(ex.map(_rtz_chunk, [(fmt, c * chunk, chunk) for c in range(64)]))
    return out


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_rtz_exhaustive_properties(rtz_sweeps, fmt):
    res = rtz_sweeps[fmt]
    assert sum(b for b, _, _, _ in res) == 0            # defining inequalities on all 2^32
    assert sum(l for _, l, _, _ in res) == 0            # lossless where the paper says it is
    assert all(ok for _, _, ok, _ in res)               # NaN -> (0x7FFF, 0)
    if fmt == "bf16":
        assert sum(t for _, _, _, t in res) == 0        # 16 extra bits = full fp32 accuracy


def test_rtz_fp16_brute_force_search(orc):
    """Independent check: the largest-magnitude finite fp16 value not above |x|, by bisection over
    the sorted list of all finite fp16 magnitudes (numpy's exact fp16 -> fp32 widening)."""
    mags = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    x = np.concatenate([(synth.normal_f32(20000, 1.0, 1, 1) * np.exp2(synth.rng(1, 2).integers(-26, 18, 20000))).astype(np.float32),
                        synth.edge_f32()]).astype(np.float32)
    x = x[np.isfinite(x)]
    idx = np.searchsorted(mags, np.abs(x.astype(np.float64)), side="right") - 1
    want = idx.astype(np.uint16) | np.where(np.signbit(x), 0x8000, 0).astype(np.uint16)
    got = np.array([orc.rtz16("fp16", int(u)) for u in x.view(np.uint32)], np.uint16)
    assert np.array_equal(got, want)


def test_mix64_uniform_and_stream_independent(orc):
    n = 1 << 16
    top = np.array([orc.mix64(0xB0B, 3, i) >> 56 for i in range(n)], np.int64)
    counts = np.bincount(top, minlength=256)
    chi2 = float(((counts - n / 256) ** 2 / (n / 256)).sum())
    assert chi2 < 256 + 5 * np.sqrt(2 * 256)            # 255 d.o.f., 5 sigma
    a = [orc.mix64(1, 0, i) for i in range(64)]
    b = [orc.mix64(1, 1, i) for i in range(64)]
    c = [orc.mix64(2, 0, i) for i in range(64)]
    assert len(set(a) & set(b)) == 0 and len(set(a) & set(c)) == 0


def test_sr_neighbours_and_closed_forms(orc):
    x = np.concatenate([(synth.normal_f32(4000, 1.0, 7, 1) * np.exp2(synth.rng(7, 2).integers(-20, 15, 4000))).astype(np.float32),
                        synth.edge_f32()]).astype(np.float32)
    for u in x.view(np.uint32):
        u = int(u)
        if _nan32(np.uint32(u)) or (u & 0x7FFFFFFF) >= 0x47800000:
            continue
        t = orc.rtz16("fp16", u)
        up = (t + 1) & 0xFFFF
        exact = orc.widen16("fp16", t) == u
        lo, hi = orc.sr16(u, 0xFFFFFFFF), orc.sr16(u, 0)
        assert lo == t                                    # the largest draw never rounds up
        assert hi == (t if exact else up)                 # the zero draw rounds up iff inexact
        assert orc.sr16(u, 0x12345678) in (t, up)


def test_sr_unbiased(orc):
    """E[widen(SR(x))] = x: 4096 draws per value, 5-sigma bound."""
    xs = np.array([1.0003, -3.14159, 1e-3, 2.5e-5, 777.77], np.float32)
    n = 4096
    for x in xs:
        h, r = orc.split_s("sr", "fp16", np.full(n, x, np.float32), seed=0xC0FFEE, stream=1)
        vals = orc.widen("fp16", h).astype(np.float64)
        t = orc.widen16("fp16", orc.rtz16("fp16", int(np.float32(x).view(np.uint32))))
        lo = np.uint32(t).view(np.float32).astype(np.float64)
        ulp = np.abs(vals - lo).max() or 1.0
        p = abs(float(x) - lo) / ulp
        sigma = ulp * np.sqrt(max(p * (1 - p), 1e-12) / n)
        assert abs(vals.mean() - float(x)) <= 5 * sigma + 1e-12 * abs(float(x))


def test_sr_reconstruct_exact_on_normal_range(orc):
    x = synth.normal_f32(1 << 18, 1.0, 11, 1) * np.float32(2.0) ** synth.rng(11, 2).integers(-13, 15, 1 << 18)
    x = x.astype(np.float32)
    x = x[(np.abs(x) >= 2.0 ** -14) & (np.abs(x) < 65504)]
    h, r = orc.split_s("sr", "fp16", x, seed=9, stream=4)
    assert np.array_equal(orc.reconstruct_s("sr", "fp16", h, r).view(np.uint32), x.view(np.uint32))
    t = np.array([orc.rtz16("fp16", int(u)) for u in x.view(np.uint32)], np.uint16)
    assert np.all((h == t) | ((h & 0x7FFF) == (t & 0x7FFF) + 1))
    assert np.all(np.abs(r.astype(np.int64)) < 8192)        # 13 extra bits + the un-round sign


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_x8_value_is_rne_and_error_bound(orc, fmt):
    x = synth.normal_f32(1 << 18, 1.0, 13, 1) * np.float32(2.0) ** synth.rng(13, 2).integers(-12, 14, 1 << 18)
    x = np.concatenate([x.astype(np.float32), synth.edge_f32()])
    h8, r8 = orc.split_s("x8", fmt, x)
    h, r = orc.split(fmt, x)
    assert np.array_equal(h8, h)
    rec = orc.reconstruct_s("x8", fmt, h8, r8).view(np.uint32).astype(np.int64)
    u = x.view(np.uint32).astype(np.int64)
    sh = 8 if fmt == "bf16" else 5
    ok = np.isfinite(x) & (np.abs(x) >= (2.0 ** -14 if fmt == "fp16" else 0)) & (np.abs(x) < 65504)
    err = np.abs(rec - u)[ok]
    sat = (np.abs(r8[ok].astype(np.int64)) >= 127)
    assert (err[~sat] <= (1 << (sh - 1))).all()
    assert (err[sat] <= (1 << sh)).all()
    d = (u - orc.widen(fmt, h).view(np.uint32).astype(np.int64))[ok]
    assert (err[((d % (1 << sh)) == 0) & ~sat] == 0).all()   # representable extra bits are exact


def _master_adam(w, gs_list, **hp):
    m = np.zeros_like(w); v = np.zeros_like(w)
    for t, g in enumerate(gs_list, start=1):
        oracle.adam_step_master("fp32", w, g, m, v, step=t, **hp)
    return w


def test_bf16_rtz_adam_equals_fp32_master(orc):
    """Lossless bf16 RTZ storage: 60 AdamW steps bit-identical to the fp32 master on every element."""
    n = 1 << 15
    w = synth.weights(n, 0.02, 0xB0B)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, adamw=True)
    grads = [orc.widen("bf16", synth.grads(n, 1e-3, "bf16", 0xB0B, t)) for t in range(1, 61)]
    master = _master_adam(w.copy(), grads, **hp)
    h, r = orc.split_s("rtz", "bf16", w)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    for t, g in enumerate(grads, start=1):
        orc.adam_step_s("rtz", "bf16", "fp32", h, r, g, m, v, step=t, **hp)
    assert np.array_equal(orc.reconstruct_s("rtz", "bf16", h, r).view(np.uint32), master.view(np.uint32))


def test_fp16_sr_adam_equals_master_where_storage_exact(orc):
    n = 1 << 15
    w = synth.weights(n, 0.02, 2023)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, adamw=False)
    grads = [orc.widen("fp16", synth.grads(n, 1e-3, "fp16", 2023, t)) for t in range(1, 41)]
    wm = w.copy(); m0 = np.zeros(n, np.float32); v0 = np.zeros(n, np.float32)
    small = np.abs(wm) < 2.0 ** -15
    h, r = orc.split_s("sr", "fp16", w, seed=1, stream=0)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    for t, g in enumerate(grads, start=1):
        orc.adam_step_master("fp32", wm, g, m0, v0, step=t, **hp)
        small |= np.abs(wm) < 2.0 ** -15
        orc.adam_step_s("sr", "fp16", "fp32", h, r, g, m, v, step=t, seed=1000 + t, stream=0, **hp)
    got = orc.reconstruct_s("sr", "fp16", h, r)
    assert np.array_equal(got.view(np.uint32)[~small], wm.view(np.uint32)[~small])
    assert small.sum() < n // 10     # ~4 % of N(0, 0.02) weights pass near zero in 40 steps


def test_x8_adam_drift_bounded(orc):
    """Each split keeps the weight within half a kept quantum (2^4 binary32 ulps for fp16+8) and the
    update does not feed the weight error back (Adam's m, v depend on the grads only), so after T
    steps |w - w_master| <= (T + 1) * 2^4 * ulp32(max_t |w_t|) (the P6-style bound)."""
    n = 1 << 14
    fmt = "fp16"
    w = synth.weights(n, 0.02, 3)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, adamw=False)
    T = 20
    grads = [orc.widen(fmt, synth.grads(n, 1e-3, fmt, 3, t)) for t in range(1, T + 1)]
    wm = w.copy(); m0 = np.zeros(n, np.float32); v0 = np.zeros(n, np.float32)
    wmax = np.abs(wm).copy()
    wmin = np.abs(wm).copy()
    h, r = orc.split_s("x8", fmt, w)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    for t, g in enumerate(grads, start=1):
        orc.adam_step_master("fp32", wm, g, m0, v0, step=t, **hp)
        wmax = np.maximum(wmax, np.abs(wm))
        wmin = np.minimum(wmin, np.abs(wm))
        orc.adam_step_s("x8", fmt, "fp32", h, r, g, m, v, step=t, **hp)
    got = orc.reconstruct_s("x8", fmt, h, r).astype(np.float64)
    ulp = np.spacing(np.maximum(wmax, 2.0 ** -14).astype(np.float32)).astype(np.float64)
    normal = wmin >= 2.0 ** -14     # fp16 subnormal range: the kept bits cannot reach (R5, R14)
    assert (np.abs(got - wm) <= (T + 1) * 16 * ulp)[normal].all()
    assert (np.abs(got - wm) <= (T + 1) * 2.0 ** -24)[~normal].all()
    assert np.array_equal(m, m0) and np.array_equal(v, v0)   # the state never sees the storage error


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_x8z_is_significand_truncation(orc, fmt):
    """keeping only the first part of the fp32 significand is round-to-zero; with 8 extra bits
    ("fp16+8") split + reconstruct clears the low 8 (bf16) / 5 (fp16: 13 - 8) bits of the
    binary32 pattern -- where the kept field can hold the remainder (bf16: every finite value;
    fp16: the normal range [2^-14, 65504]) -- the value is the RTZ value, the code is the next 8
    bits, and NaN / Inf store no extra bits."""
    hi = np.arange(1 << 16, dtype=np.uint32) << 16
    lo = synth.rng(21, 1).integers(0, 1 << 16, size=(1 << 16, 64), dtype=np.uint32)
    u = (hi[:, None] | lo).reshape(-1)
    x = u.view(np.float32)
    h, r = orc.split_s("x8z", fmt, x)
    assert r.dtype == np.uint8
    ht = np.array([orc.rtz16(fmt, int(v)) for v in u[::997]], np.uint16)
    assert np.array_equal(h[::997], ht)                                # the value is RTZ (pinned above)
    rec = orc.reconstruct_s("x8z", fmt, h, r).view(np.uint32)
    sh = 8 if fmt == "bf16" else 5
    a = u & 0x7FFFFFFF
    fin = a < 0x7F800000
    if fmt == "bf16":
        ok = fin & (np.abs(x) <= np.float32(3.3895314e38))             # RTZ saturates above bf16 max
    else:
        ok = fin & (a >= 0x38800000) & (np.abs(x) < 65520)             # fp16 normal range
    assert np.array_equal(rec[ok], u[ok] & ~np.uint32((1 << sh) - 1))
    # everywhere (saturated codes included) the stored weight is a truncation: never larger in
    # magnitude, never of the other sign
    assert (_mag(rec[fin]) <= _mag(u[fin])).all()
    assert ((rec[fin] ^ u[fin]) & 0x80000000 == 0)[_mag(rec[fin]) != 0].all()
    nan = a > 0x7F800000
    assert (h[nan] == 0x7FFF).all() and not r[nan].any()
    inf = a == 0x7F800000
    assert not r[inf].any() and np.isinf(orc.reconstruct_s("x8z", fmt, h[inf], r[inf])).all()


def test_x8z_adam_error_is_truncation(orc):
    """fp16+8 (truncated) Adam: every split rounds the weight toward zero by less than one kept
    quantum (2^5 binary32 ulps), so after T steps the weight lies within (T + 1) quanta of the
    fp32 master and the state (m, v) never sees the storage error."""
    n = 1 << 14
    fmt = "fp16"
    w = synth.weights(n, 0.02, 5)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, adamw=False)
    T = 20
    grads = [orc.widen(fmt, synth.grads(n, 1e-3, fmt, 5, t)) for t in range(1, T + 1)]
    wm = w.copy(); m0 = np.zeros(n, np.float32); v0 = np.zeros(n, np.float32)
    wmax, wmin = np.abs(wm).copy(), np.abs(wm).copy()
    h, r = orc.split_s("x8z", fmt, w)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    for t, g in enumerate(grads, start=1):
        orc.adam_step_master("fp32", wm, g, m0, v0, step=t, **hp)
        wmax, wmin = np.maximum(wmax, np.abs(wm)), np.minimum(wmin, np.abs(wm))
        orc.adam_step_s("x8z", fmt, "fp32", h, r, g, m, v, step=t, **hp)
    got = orc.reconstruct_s("x8z", fmt, h, r).astype(np.float64)
    ulp = np.spacing(np.maximum(wmax, 2.0 ** -14).astype(np.float32)).astype(np.float64)
    normal = wmin >= 2.0 ** -14
    assert (np.abs(got - wm) <= (T + 1) * 32 * ulp)[normal].all()
    assert np.array_equal(m, m0) and np.array_equal(v, v0)
