"""Helpers shared by the GPU parity tests: numpy <-> CUDA tensor marshalling of bit patterns.
(No method arithmetic here.)"""
import numpy as np
import torch

TDT = {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}


def dev16(bits: np.ndarray, fmt: str) -> torch.Tensor:
    """uint16 bit patterns -> CUDA tensor of dtype fmt (bit-identical)."""
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16).copy()).view(TDT[fmt]).cuda()


def host16(t: torch.Tensor) -> np.ndarray:
    return t.detach().view(torch.int16).cpu().numpy().view(np.uint16)


def dev_grad(g: np.ndarray, gfmt: str) -> torch.Tensor:
    if gfmt == "fp32":
        return torch.from_numpy(np.ascontiguousarray(g, dtype=np.float32).copy()).cuda()
    return dev16(g, gfmt)


def devf(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32).copy()).cuda()


def devi16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int16).copy()).cuda()


def hostf(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy() if t.dtype != torch.float32 else t.detach().cpu().numpy()


def bits32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def same_bits_nan_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """fp32 arrays bit-identical, except that any NaN equals any NaN (NaN payloads of the fp32
    optimizer state are not specified: x86 propagates an operand's payload, the GPU a canonical
    NaN; R4)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb) and np.array_equal(a.view(np.uint32)[~na], b.view(np.uint32)[~nb]))


def ordered16(h: np.ndarray, fmt: str) -> np.ndarray:
    """Map 16-bit float patterns to integers monotone in value (for ulp distances)."""
    h = h.astype(np.int64)
    mag = h & 0x7FFF
    return np.where(h & 0x8000, -mag, mag)


def ulp16_dist(a: np.ndarray, b: np.ndarray, fmt: str) -> np.ndarray:
    return np.abs(ordered16(a, fmt) - ordered16(b, fmt))
