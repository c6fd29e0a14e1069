"""Diagnostic (GPU): replicate tests/test_gpu_parity.py::test_gpt2_adamw_full[False] and dump failures."""
import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle, synth
import paper_2309_12381_b200 as mpo
import test_gpu_parity as T
from gpu_util import dev16, devi16, devf, host16
oracle.build()
fmt = "bf16"
sizes, h, r, g, m, v = T._workload_table(mpo, "gpt2_small", fmt, "adam", 2023)
V = T._aligned_copy(lambda a: dev16(a, fmt), h, sizes); R = T._aligned_copy(devi16, r, sizes)
G = T._aligned_copy(lambda a: dev16(a, fmt), g, sizes); M = T._aligned_copy(devf, m, sizes); W = T._aligned_copy(devf, v, sizes)
hp = mpo.AdamParams(lr=6e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, adamw=True, step=5)
pre = (h.copy(), r.copy(), m.copy(), v.copy())
mpo.mpo_adam_step(mpo.TensorTable(V, R, G, M, W), hp, exact=False)
oracle.adam_step(fmt, fmt, h, r, g, m, v, **T._adam_hp_kw(hp))
hg = np.concatenate([host16(x) for x in V]); rg = np.concatenate([x.cpu().numpy() for x in R])
mg = np.concatenate([x.cpu().numpy() for x in M]); vg = np.concatenate([x.cpu().numpy() for x in W])
wg = oracle.reconstruct(fmt, hg, rg).astype(np.float64); wo = oracle.reconstruct(fmt, h, r).astype(np.float64)
w0 = oracle.reconstruct(fmt, pre[0], pre[1]).astype(np.float64)
g32 = oracle.widen(fmt, g)
us = T._adam_uscale(hp, pre[2], g32, v)
err = np.abs(wg - wo); bound = 1e-6 * (np.abs(w0) + np.abs(wo)) + 1e-6 * us
bad = np.nonzero(err > bound)[0]
print("n bad", len(bad), "tensor offsets", np.cumsum([0] + sizes)[:5])
for i in bad[:12]:
    print("i", i, "w0 %.9g g %.6g m0 %.6g v0 %.6g | wo %.9g wg %.9g err %.3g bound %.3g us %.3g | mo %.6g mg %.6g vo %.6g vg %.6g | ho %04x hg %04x ro %d rg %d"
          % (w0[i], g32[i], pre[2][i], pre[3][i], wo[i], wg[i], err[i], bound[i], us[i], m[i], mg[i], v[i], vg[i], h[i], hg[i], r[i], rg[i]))
