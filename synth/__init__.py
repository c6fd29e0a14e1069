"""Seeded synthetic input generators shared by the oracle tests, the GPU parity tests and
bench.py.  This module holds NONE of the method's arithmetic (no split, reconstruct or
update): it draws random fp32 weights and 16-bit gradients (a 16-bit gradient is produced by
the library cast of numpy / torch, as a training framework would hand it over), plus the
edge-case vectors of SURVEY.md 8(d) C1.

Input recipe:
* weights  w ~ N(0, 0.02) fp32 (GPT/LLaMA-style init; ResNet conv Kaiming fan-out is in the
  same range), seed 0xB0B unless stated;
* gradients g_t ~ N(0, sigma_g) cast to the value format (fp16 / bf16) or kept fp32, one
  independent stream per (seed, step);
* the paper's seeds: 0xB0B, 2023, 0xC0FFEE.
"""
from __future__ import annotations

import numpy as np

SEEDS = (0xB0B, 2023, 0xC0FFEE)

FP16, BF16, FP32 = "fp16", "bf16", "fp32"


def rng(seed: int, *stream: int) -> np.random.Generator:
    """Counter-based Philox generator keyed by (seed, stream...)."""
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([int(seed)] + [int(s) for s in stream])))


def normal_f32(n: int, std: float, seed: int, *stream: int) -> np.ndarray:
    return (rng(seed, *stream).standard_normal(n, dtype=np.float32) * np.float32(std)).astype(np.float32)


def to16_bits(x: np.ndarray, fmt: str) -> np.ndarray:
    """Library cast of fp32 to a 16-bit format, returned as uint16 bit patterns.

    fp16: numpy's IEEE cast; bf16: torch's CPU cast.  Only used to MAKE 16-bit gradient
    inputs; the method's own rounding lives in oracle/ and in the CUDA kernels."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if fmt == FP16:
        return x.astype(np.float16).view(np.uint16)
    if fmt == BF16:
        import torch
        return torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    raise ValueError(fmt)


def grads(n: int, std: float, fmt: str, seed: int, step: int) -> np.ndarray:
    """Gradient of step ``step``: N(0, std) fp32, delivered in ``fmt`` (uint16 bits for
    fp16/bf16, float32 for fp32)."""
    g = normal_f32(n, std, seed, 1, step)
    if fmt == FP32:
        return g
    return to16_bits(g, fmt)


def weights(n: int, std: float = 0.02, seed: int = 0xB0B) -> np.ndarray:
    return normal_f32(n, std, seed, 0, 0)


def edge_f32() -> np.ndarray:
    """Edge-case fp32 values: signed zeros, fp32 and fp16 subnormals,
    exact RNE ties of both formats, the fp16 overflow boundary 65504/65520, tiny |x| < 2^-17,
    the bf16 overflow boundary, +-Inf and NaN."""
    u = [
        0x00000000, 0x80000000,                      # +-0
        0x00000001, 0x807FFFFF, 0x00400000,          # fp32 subnormals
        0x3F808000, 0x3F818000, 0x3F80C000,          # bf16 ties / halfway (P4)
        0x3F801000, 0x3F803000, 0x3F800800,          # fp16 ties around 1.0
        0x477FE000, 0x477FEFFF, 0x477FF000, 0x477FF001,   # 65504, <65520, 65520 (tie), >65520
        0xC77FF000,                                  # -65520
        0x33800000, 0x33000000, 0x33C00000,          # 2^-24, 2^-25, 1.5*2^-24
        0x37800000, 0x37000000, 0x37000001, 0x36800000,   # 2^-16, 2^-17, 2^-17+, 2^-18
        0x387FC000, 0x38800000,                      # fp16 subnormal/normal boundary
        0x7F7F8000, 0x7F7F7FFF, 0x7F7FFFFF,          # bf16 overflow boundary
        0x7F800000, 0xFF800000,                      # +-Inf
        0x7FC00000, 0xFFC00001, 0x7F800001,          # NaNs
        0x3F800000, 0xBF800000, 0x3FC00000,          # 1, -1, 1.5
    ]
    return np.array(u, dtype=np.uint32).view(np.float32)


def torch_normal_(t, std: float, seed: int, stream: int = 0):
    """Fill a (device) torch tensor with N(0, std) from a seeded torch generator (bench and
    full-size GPU tests; the oracle checks sampled windows copied from the same tensor)."""
    import torch
    g = torch.Generator(device=t.device)
    g.manual_seed((seed * 1_000_003 + stream) & 0x7FFFFFFFFFFFFFFF)
    if t.dtype in (torch.float16, torch.bfloat16):
        # draw in fp32 chunks and let torch cast (library cast, round-to-nearest-even)
        flat = t.view(-1)
        chunk = 1 << 28
        for i in range(0, flat.numel(), chunk):
            part = flat[i:i + chunk]
            tmp = torch.empty(part.numel(), dtype=torch.float32, device=t.device)
            tmp.normal_(0.0, std, generator=g)
            part.copy_(tmp)
            del tmp
        return t
    return t.normal_(0.0, std, generator=g)
