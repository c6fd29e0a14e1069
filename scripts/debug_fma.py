"""Diagnostic (GPU): dump inputs of elements where the FMA build leaves the tolerance, GPT-2 recipe."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle, synth
import paper_2309_12381_b200 as mpo
from paper_2309_12381_b200 import api
from gpu_util import dev16, devi16, devf, host16
oracle.build()
print("selfcheck", api.mpo_selfcheck_fastmath(pairs=1 << 31, seed=0xC0FFEE))
fmt = "bf16"; n = 1 << 22; seed = 2023
w = synth.weights(n, 0.02, seed); h, r = oracle.split(fmt, w)
g = synth.grads(n, 1e-3, fmt, seed, 1)
m = synth.normal_f32(n, 1e-4, seed, 3); v = np.abs(synth.normal_f32(n, 1e-7, seed, 4))
hp = mpo.AdamParams(lr=6e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, adamw=True, step=5)
res = {}
for exact in (False, True):
    V, R, G, M, W = dev16(h, fmt), devi16(r), dev16(g, fmt), devf(m), devf(v)
    mpo.mpo_adam_step(mpo.TensorTable([V], [R], [G], [M], [W]), hp, exact=exact)
    res[exact] = (host16(V), R.cpu().numpy(), M.cpu().numpy(), W.cpu().numpy())
ho, ro, mo, vo = h.copy(), r.copy(), m.copy(), v.copy()
oracle.adam_step(fmt, fmt, ho, ro, g, mo, vo, lr=6e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, adamw=True, step=5)
wo = oracle.reconstruct(fmt, ho, ro).astype(np.float64)
w0 = oracle.reconstruct(fmt, h, r).astype(np.float64)
for exact in (False, True):
    hg, rg, mg, vg = res[exact]
    wg = oracle.reconstruct(fmt, hg, rg).astype(np.float64)
    err = np.abs(wg - wo); u = np.abs(w0 * (1 - 6e-4 * 0.1) - wo)
    rel = err / np.maximum(u, 1e-30)
    idx = np.argsort(-rel)[:6]
    print("exact" if exact else "fma", "max err", err.max(), "n(err>0)", int((err > 0).sum()), "max err/u", rel.max())
    print("  m diff", int((mg != mo).sum()), "v diff", int((vg != vo).sum()))
    for i in idx:
        print("   i", i, "w0", w0[i], "g", oracle.widen(fmt, g[i:i+1])[0], "m0", m[i], "v0", v[i], "wo", wo[i], "wg", wg[i],
              "mo", mo[i], "mg", mg[i], "vo", vo[i], "vg", vg[i])
