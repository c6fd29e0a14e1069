"""Fig. rstoc of the paper ("Forward Error On 16bits Tensor Addition"), reproduced
through this library's GPU step: the in-place addition w <- w + b of standard-normal tensors
("operations with random values following the standard normal distribution"), run as the
residual-compensated SGD step with lr = -1, no momentum, no decay, on fp16 values under every
storage scheme, next to classical fp16 (torch, no extra bits) and fp32 (torch).

  * single operation vs tensor size n: a ~ N(0,1) stored in the format, b ~ N(0,1) rounded to
    fp16 (the same exact operand for every variant), one addition;
  * cumulative: K successive additions of fresh N(0,1) tensors (n = 2^20), error after K
    operations, and the mean condition number sum|x_k| / |sum x_k| of the element sums.

Error = ||reconstruct(result) - exact||_2 / ||exact||_2, exact = the fp64 sum of the stored
initial value and the operands; `bias` = mean signed error / mean |exact|.  Stochastic rounding
draws a fresh key per operation (api.step_seed).
usage: python scripts/error_bench.py > profiles/r02_error_bench.jsonl"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCHEMES = ("rne", "rtz", "sr", "x8", "x8z")   # fp16 + 16-bit residual (RNE / RTZ / SR), fp16 + 8 bits (RNE / RTZ)


def _stored(mpo, w32, scheme, seed):
    v, r = mpo.mpo_split(w32, torch.float16, scheme=scheme, seed=seed, sr_stream=0)
    return v, r


def accumulate(mpo, a32, bs, scheme, seed=1234):
    """Stores a32 under `scheme`, adds every tensor of `bs` (fp16) in place with the library's SGD
    step (lr = -1); returns (fp32 result, fp64 exact sum of the stored start and the operands)."""
    from paper_2309_12381_b200 import api
    v, r = _stored(mpo, a32, scheme, seed)
    exact = mpo.mpo_reconstruct(v, r, scheme=scheme).double()
    tab = mpo.TensorTable([v], [r], [bs[0]], [None], [None], scheme=scheme)
    for k, b in enumerate(bs):
        tab.set_grads([b])
        mpo.mpo_sgd_step(tab, mpo.SgdParams(lr=-1.0, seed=api.step_seed(seed, k + 1)))
        exact += b.double()
    return mpo.mpo_reconstruct(v, r, scheme=scheme).double(), exact


def _metrics(got, exact):
    err = got - exact
    return {"rel_err": float(err.norm() / exact.norm()),
            "bias": float(err.mean() / exact.abs().mean())}


def single_op(mpo, n, gen):
    a = torch.randn(n, device="cuda", generator=gen)
    b = torch.randn(n, device="cuda", generator=gen).half()
    out = {}
    a16 = a.half()
    out["fp16"] = _metrics((a16 + b).double(), a16.double() + b.double())     # classical: both fp16
    out["fp32"] = _metrics((a + b.float()).double(), a.double() + b.double())
    for s in SCHEMES:
        got, exact = accumulate(mpo, a, [b], s)
        out[f"fp16+{s}"] = _metrics(got, exact)
    return out


def cumulative(mpo, n, K, gen):
    a = torch.randn(n, device="cuda", generator=gen)
    bs = [torch.randn(n, device="cuda", generator=gen).half() for _ in range(K)]
    out = {}
    a16 = a.half()
    acc16, acc32 = a16.clone(), a.clone()
    for b in bs:
        acc16 += b
        acc32 += b.float()
    ex16 = a16.double() + sum(b.double() for b in bs)
    ex32 = a.double() + sum(b.double() for b in bs)
    out["fp16"] = _metrics(acc16.double(), ex16)
    out["fp32"] = _metrics(acc32.double(), ex32)
    for s in SCHEMES:
        got, exact = accumulate(mpo, a, bs, s)
        out[f"fp16+{s}"] = _metrics(got, exact)
    absum = a.double().abs() + sum(b.double().abs() for b in bs)
    out["condition_number_mean"] = float((absum / ex32.abs().clamp_min(1e-30)).clamp_max(1e12).mean())
    return out


def main():
    import paper_2309_12381_b200 as mpo
    from paper_2309_12381_b200 import _build
    _build.build()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2023)
    for e in range(2, 8):
        print(json.dumps({"experiment": "single_op", "n": 10 ** e, **single_op(mpo, 10 ** e, gen)}), flush=True)
    for K in (1, 10, 100, 1000, 10000):
        print(json.dumps({"experiment": "cumulative", "n": 1 << 20, "ops": K,
                          **cumulative(mpo, 1 << 20, K, gen)}), flush=True)


if __name__ == "__main__":
    main()
