"""Pins of the oracle's number formats, split and reconstruct (no GPU).

Each check ties oracle/oracle.c to something other than itself:
* P1  exhaustive 2^16 sweep: every exactly representable 16-bit value splits to a zero residual
      and reconstructs bit-identically (BASELINE north_star; "13 and 16 bits of precision
      to keep if we want to maintain a full fp32 accuracy").
* P3  library routine: the oracle's RNE equals torch's CPU float32->float16 (F16C hardware
      conversion) and float32->bfloat16 casts on ALL 2^32 binary32 patterns (NaN excepted,
      reading R4), numpy's float16 cast on sampled patterns, and the oracle's widening equals
      numpy/torch widening on all 2^16 patterns.
* P2  closed-form loss counts of the int16 residual (reading R3) over all 2^32 patterns.
* P4  worked examples (tests/golden/split_examples.txt, each row cited).
"""
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "split_examples.txt")


def _nan32(u):
    return (u & 0x7FFFFFFF) > 0x7F800000


# ----------------------------------------------------------------------------------- P1 --
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_p1_exhaustive_16bit_roundtrip(orc, fmt):
    h = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    w = orc.widen(fmt, h)
    wu = w.view(np.uint32)
    nan = _nan32(wu)
    h2, r2 = orc.split(fmt, w)
    # exactly representable -> same 16-bit pattern, zero residual
    assert np.array_equal(h2[~nan], h[~nan])
    assert not r2[~nan].any()
    # reconstruct is bit-identical to the widened value
    assert np.array_equal(orc.reconstruct(fmt, h2, r2).view(np.uint32)[~nan], wu[~nan])
    # NaN patterns -> canonical (0x7FFF, 0) (R4)
    assert (h2[nan] == 0x7FFF).all() and not r2[nan].any()
    expected_nan = 2 * (2 ** 10 - 1) if fmt == "fp16" else 2 * (2 ** 7 - 1)
    assert nan.sum() == expected_nan


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_p3_widen_matches_library(orc, fmt):
    import torch
    h = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    ours = orc.widen(fmt, h).view(np.uint32)
    if fmt == "fp16":
        lib = h.view(np.float16).astype(np.float32).view(np.uint32)
    else:
        lib = torch.from_numpy(h.view(np.int16)).view(torch.bfloat16).float().numpy().view(np.uint32)
    nan = _nan32(lib)
    assert np.array_equal(ours[~nan], lib[~nan])
    assert (ours[nan] == 0x7FFFFFFF).all()


# ------------------------------------------------------------------------------ P2 / P3 --
def _sweep_chunk(args):
    """One 2^26-pattern chunk: library-cast mismatches and residual-loss statistics."""
    fmt, lo, n = args
    import torch
    torch.set_num_threads(1)
    oracle.lib()
    u = np.arange(lo, lo + n, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    a = u & np.uint32(0x7FFFFFFF)
    nan = a > 0x7F800000
    h, r = oracle.split(fmt, x)
    tdt = torch.float16 if fmt == "fp16" else torch.bfloat16
    lib = torch.from_numpy(x).to(tdt).view(torch.int16).numpy().view(np.uint16)
    ok = nan | (h == lib)
    mism = int(n - np.count_nonzero(ok))
    nan_ok = bool((h[nan] == 0x7FFF).all() and not r[nan].any())
    rec = oracle.reconstruct(fmt, h, r).view(np.uint32)
    inf_pat = 0x7C00 if fmt == "fp16" else 0x7F80
    inf = ((h & 0x7FFF) == inf_pat) & ~nan
    lossy = (rec != u) & ~nan & ~inf
    ul = u[lossy]
    al = ul & np.uint32(0x7FFFFFFF)
    err = np.abs(ul.view(np.float32).astype(np.float64) - rec[lossy].view(np.float32).astype(np.float64))
    # lossy counts by magnitude band (fp16 closed forms; bounds as binary32 patterns)
    bands = {}
    for name, lo_b, hi_b in [("ge_2m16", 0x37800000, 0x477FF000), ("2m17_2m16", 0x37000000, 0x37800000),
                             ("2m18_2m17", 0x36800000, 0x37000000)]:
        bands[name] = int(np.count_nonzero((al >= lo_b) & (al < hi_b)))
    bf16_struct = int(np.count_nonzero(((ul & 0xFFFF) != 0x8000) | (((ul >> 16) & 1) != 0)))
    one_ulp_low = bool(((ul - rec[lossy]) == 1).all()) if fmt == "bf16" else True
    return dict(mism=mism, nan_ok=nan_ok, nan=int(nan.sum()), inf=int(inf.sum()),
                lossy=int(lossy.sum()), maxerr=float(err.max()) if err.size else 0.0,
                bands=bands, bf16_struct=bf16_struct, one_ulp_low=one_ulp_low)


@pytest.fixture(scope="module")
def sweeps(orc):
    chunk = 1 << 26
    out = {}
    import multiprocessing as mp
    ctx = mp.get_context("spawn")      # no fork after torch/OpenMP initialisation
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1), mp_context=ctx) as ex:
        for fmt in ("fp16", "bf16"):
            parts = list(ex.map(_sweep_chunk, [(fmt, lo, chunk) for lo in range(0, 1 << 32, chunk)]))
            agg = dict(mism=0, nan=0, inf=0, lossy=0, maxerr=0.0, bf16_struct=0,
                       nan_ok=True, one_ulp_low=True, bands={})
            for p in parts:
                for k in ("mism", "nan", "inf", "lossy", "bf16_struct"):
                    agg[k] += p[k]
                agg["maxerr"] = max(agg["maxerr"], p["maxerr"])
                agg["nan_ok"] &= p["nan_ok"]
                agg["one_ulp_low"] &= p["one_ulp_low"]
                for k, v in p["bands"].items():
                    agg["bands"][k] = agg["bands"].get(k, 0) + v
            out[fmt] = agg
    return out


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_p3_rne_matches_library_on_all_2_32(sweeps, fmt):
    s = sweeps[fmt]
    assert s["mism"] == 0
    assert s["nan_ok"]
    assert s["nan"] == 2 * (2 ** 23 - 1)


def test_p2_bf16_loss_closed_form(sweeps):
    s = sweeps["bf16"]
    # lossy exactly when the dropped half is 0x8000 and the kept half is even (the RNE tie
    # rounded down gives +32768, which saturates to +32767, R3): per sign 255 finite
    # exponents x 64 even 7-bit mantissas.
    assert s["lossy"] == 2 * 255 * 64 == 32640
    assert s["bf16_struct"] == 0
    assert s["one_ulp_low"]
    # overflow to Inf: [0x7F7F8000, 0x7F7FFFFF] per sign (2 x 32768) plus the two Infs ... the
    # two real Infs are inside the count of patterns whose value16 is Inf.
    assert s["inf"] == 2 * 32768 + 2


def test_p2_fp16_loss_closed_form(sweeps):
    s = sweeps["fp16"]
    b = s["bands"]
    # |x| >= 2^-16: half an fp16 quantum is at most 2^13 (normal) / 2^14 (subnormal) ulp32
    assert b["ge_2m16"] == 0
    # [2^-17, 2^-16): half-quantum = 2^15 ulp32; only ties rounded down to an even subnormal
    # are lossy: 64 per sign (k = 128..255 even)
    assert b["2m17_2m16"] == 2 * 64
    # [2^-18, 2^-17): quantum = 2^17 ulp32; exactly half of each quantum fits int16
    assert b["2m18_2m17"] == 2 * 2 ** 22
    # any saturated residual is at most half an fp16 subnormal quantum away: 2^-25
    assert s["maxerr"] == 2.0 ** -25
    # |x| >= 65520 rounds to Inf (IEEE): per sign exponents 143..254 (112 x 2^23) plus
    # [65520, 65536) (0x1000 patterns) plus the Inf itself
    assert s["inf"] == 2 * (112 * 2 ** 23 + 0x1000 + 1)


# ----------------------------------------------------------------------------------- P4 --
def _golden():
    rows = []
    for line in open(GOLDEN):
        line = line.split("#", 1)[0].strip() if line.startswith("#") else line.strip()
        if not line:
            continue
        f = line.split()
        rows.append((f[0], int(f[1], 16), int(f[2], 16), int(f[3]), int(f[4], 16)))
    return rows


@pytest.mark.parametrize("row", _golden(), ids=lambda r: f"{r[0]}-{r[1]:08x}")
def test_p4_worked_examples(orc, row):
    fmt, xin, hv, rv, rec = row
    x = np.array([xin], np.uint32).view(np.float32)
    h, r = orc.split(fmt, x)
    assert (int(h[0]), int(r[0])) == (hv, rv)
    assert int(orc.reconstruct(fmt, h, r).view(np.uint32)[0]) == rec


# ------------------------------------------------------------------------ invariants -----
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_split_invariants_random(orc, fmt):
    import synth
    u = synth.rng(0xB0B, 7).integers(0, 1 << 32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    nan = _nan32(u)
    h, r = orc.split(fmt, x)
    rec = orc.reconstruct(fmt, h, r)
    # idempotence: split(reconstruct(split(x))) == split(x)
    h2, r2 = orc.split(fmt, rec)
    assert np.array_equal(h2, h) and np.array_equal(r2, r)
    # the value is the RNE cast; sign preserved; reconstruct error below half an fp16/bf16 ulp
    fin = ~nan & np.isfinite(orc.widen(fmt, h))
    assert np.array_equal(np.signbit(x[fin]), np.signbit(rec[fin]))
    xd, rd = x[fin].astype(np.float64), rec[fin].astype(np.float64)
    tol = 2.0 ** -25 if fmt == "fp16" else 0.0
    rel = np.abs(xd - rd) <= np.maximum(np.abs(xd) * 2.0 ** -23, tol)
    assert rel.all()


def test_p3_rne_matches_numpy_fp16_sampled(orc):
    import synth
    u = synth.rng(0xB0B, 9).integers(0, 1 << 32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    nan = _nan32(u)
    ours = orc.cast16("fp16", x)
    assert np.array_equal(ours[~nan], x[~nan].astype(np.float16).view(np.uint16))


def test_fp16_lossless_on_normal_range(orc):
    # SPEC S:113 / P:68: fp16 + 13 extra bits is the identity on fp16's normal range
    import synth
    g = synth.rng(0xB0B, 8)
    e = g.integers(127 - 14, 127 + 16, size=1 << 20).astype(np.uint32)
    m = g.integers(0, 1 << 23, size=1 << 20).astype(np.uint32)
    s = g.integers(0, 2, size=1 << 20).astype(np.uint32)
    u = (s << 31) | (e << 23) | m
    x = u.view(np.float32)
    x = x[np.abs(x) < 65520]
    h, r = orc.split("fp16", x)
    assert np.array_equal(orc.reconstruct("fp16", h, r).view(np.uint32), x.view(np.uint32))
