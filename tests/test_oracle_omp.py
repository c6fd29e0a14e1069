"""The all-core oracle build (gcc -fopenmp, bench.py's cpu_baseline "threads_all") is the same
program: its element loops are split across threads and nothing else changes, so every output is
bit-identical to the plain single-thread build (the method is elementwise)."""
import numpy as np
import pytest

import synth


@pytest.fixture
def par(orc):
    yield orc
    orc.parallel(False)


def _run(orc, on):
    n = (1 << 20) + 13
    out = {}
    orc.parallel(on, 0)
    w = np.concatenate([synth.weights(n - 36, 0.05, 1), synth.edge_f32()]).astype(np.float32)
    for fmt in ("fp16", "bf16"):
        h, r = orc.split(fmt, w)
        out[f"split_{fmt}"] = (h, r, orc.reconstruct(fmt, h, r))
        g = synth.grads(n, 1e-2, fmt, 2, 3)
        m = synth.normal_f32(n, 1e-3, 3, 1); v = np.abs(synth.normal_f32(n, 1e-5, 3, 2))
        hh, rr = h.copy(), r.copy()
        orc.adam_step(fmt, fmt, hh, rr, g, m, v, lr=1e-3, weight_decay=0.1, step=4)
        out[f"adam_{fmt}"] = (hh, rr, m, v)
        hh, rr, b = h.copy(), r.copy(), synth.normal_f32(n, 1e-3, 4, 1)
        orc.sgd_step(fmt, fmt, hh, rr, g, b, lr=0.1, momentum=0.9, weight_decay=1e-4)
        out[f"sgd_{fmt}"] = (hh, rr, b)
    for scheme, fmt in (("sr", "fp16"), ("x8", "bf16"), ("rtz", "fp16")):
        h, r = orc.split_s(scheme, fmt, w, seed=5, stream=2)
        g = synth.grads(n, 1e-2, fmt, 2, 4)
        m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
        orc.adam_step_s(scheme, fmt, fmt, h, r, g, m, v, lr=1e-3, step=1, seed=9, stream=2)
        out[f"{scheme}_{fmt}"] = (h, r, m, v)
    return out


def test_openmp_build_is_bit_identical(par):
    seq = _run(par, False)
    threads = par.parallel(True, 0)
    assert threads >= 1
    assert par.fpenv_ok()
    mt = _run(par, True)
    for k in seq:
        for a, b in zip(seq[k], mt[k]):
            a = np.ascontiguousarray(a); b = np.ascontiguousarray(b)
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), k
