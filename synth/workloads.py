"""Parameter-shape sets of the BASELINE.json workloads (shapes only; no method arithmetic).

Shared by tests/ and bench.py.  The optimizer path only sees a list of tensor sizes, so a
workload here is the ordered list of parameter shapes of the named architecture in its
standard layout:

* ``resnet50``  torchvision ``resnet50()``: 25 557 032 params, 161 tensors (BJ configs[1]).
* ``gpt2_small`` HF GPT-2 small with tied lm_head: 124 439 808 params, 148 tensors (configs[2]).
* ``llama7b``   LLaMA-7B (untied lm_head): 6 738 415 616 params, 291 tensors (configs[3]).
* ``vit_l16``   timm ViT-L/16 224px, 1000 classes: 304 326 632 params, 296 tensors (configs[4]).
* ``flat1m``    one flat 1 048 576-element tensor (configs[0]).
"""
from __future__ import annotations

import math


def _resnet50():
    shapes = [("conv1.weight", (64, 3, 7, 7)), ("bn1.weight", (64,)), ("bn1.bias", (64,))]
    inplanes = 64
    for li, (planes, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)], start=1):
        for b in range(blocks):
            p = f"layer{li}.{b}."
            shapes += [
                (p + "conv1.weight", (planes, inplanes, 1, 1)),
                (p + "bn1.weight", (planes,)), (p + "bn1.bias", (planes,)),
                (p + "conv2.weight", (planes, planes, 3, 3)),
                (p + "bn2.weight", (planes,)), (p + "bn2.bias", (planes,)),
                (p + "conv3.weight", (planes * 4, planes, 1, 1)),
                (p + "bn3.weight", (planes * 4,)), (p + "bn3.bias", (planes * 4,)),
            ]
            if b == 0:
                shapes += [
                    (p + "downsample.0.weight", (planes * 4, inplanes, 1, 1)),
                    (p + "downsample.1.weight", (planes * 4,)),
                    (p + "downsample.1.bias", (planes * 4,)),
                ]
            inplanes = planes * 4
    shapes += [("fc.weight", (1000, 2048)), ("fc.bias", (1000,))]
    return shapes


def _gpt2_small():
    d, v, t, L = 768, 50257, 1024, 12
    shapes = [("wte.weight", (v, d)), ("wpe.weight", (t, d))]
    for i in range(L):
        p = f"h.{i}."
        shapes += [
            (p + "ln_1.weight", (d,)), (p + "ln_1.bias", (d,)),
            (p + "attn.c_attn.weight", (d, 3 * d)), (p + "attn.c_attn.bias", (3 * d,)),
            (p + "attn.c_proj.weight", (d, d)), (p + "attn.c_proj.bias", (d,)),
            (p + "ln_2.weight", (d,)), (p + "ln_2.bias", (d,)),
            (p + "mlp.c_fc.weight", (d, 4 * d)), (p + "mlp.c_fc.bias", (4 * d,)),
            (p + "mlp.c_proj.weight", (4 * d, d)), (p + "mlp.c_proj.bias", (d,)),
        ]
    shapes += [("ln_f.weight", (d,)), ("ln_f.bias", (d,))]
    return shapes


def _llama7b():
    d, ff, v, L = 4096, 11008, 32000, 32
    shapes = [("embed_tokens.weight", (v, d))]
    for i in range(L):
        p = f"layers.{i}."
        shapes += [
            (p + "self_attn.q_proj.weight", (d, d)), (p + "self_attn.k_proj.weight", (d, d)),
            (p + "self_attn.v_proj.weight", (d, d)), (p + "self_attn.o_proj.weight", (d, d)),
            (p + "mlp.gate_proj.weight", (ff, d)), (p + "mlp.up_proj.weight", (ff, d)),
            (p + "mlp.down_proj.weight", (d, ff)),
            (p + "input_layernorm.weight", (d,)), (p + "post_attention_layernorm.weight", (d,)),
        ]
    shapes += [("norm.weight", (d,)), ("lm_head.weight", (v, d))]
    return shapes


def _vit_l16():
    d, L, ff = 1024, 24, 4096
    shapes = [("cls_token", (1, 1, d)), ("pos_embed", (1, 197, d)),
              ("patch_embed.proj.weight", (d, 3, 16, 16)), ("patch_embed.proj.bias", (d,))]
    for i in range(L):
        p = f"blocks.{i}."
        shapes += [
            (p + "norm1.weight", (d,)), (p + "norm1.bias", (d,)),
            (p + "attn.qkv.weight", (3 * d, d)), (p + "attn.qkv.bias", (3 * d,)),
            (p + "attn.proj.weight", (d, d)), (p + "attn.proj.bias", (d,)),
            (p + "norm2.weight", (d,)), (p + "norm2.bias", (d,)),
            (p + "mlp.fc1.weight", (ff, d)), (p + "mlp.fc1.bias", (ff,)),
            (p + "mlp.fc2.weight", (d, ff)), (p + "mlp.fc2.bias", (d,)),
        ]
    shapes += [("norm.weight", (d,)), ("norm.bias", (d,)),
               ("head.weight", (1000, d)), ("head.bias", (1000,))]
    return shapes


WORKLOADS = {
    "flat1m": lambda: [("flat", (1 << 20,))],
    "resnet50": _resnet50,
    "gpt2_small": _gpt2_small,
    "llama7b": _llama7b,
    "vit_l16": _vit_l16,
}

EXPECTED = {  # (params, tensors), SURVEY.md 8(a)
    "flat1m": (1 << 20, 1),
    "resnet50": (25_557_032, 161),
    "gpt2_small": (124_439_808, 148),
    "llama7b": (6_738_415_616, 291),
    "vit_l16": (304_326_632, 296),
}


def shapes(name: str):
    """Ordered [(param_name, shape)] of workload ``name``."""
    return WORKLOADS[name]()


def sizes(name: str):
    return [math.prod(s) for _, s in shapes(name)]


def total(name: str) -> int:
    return sum(sizes(name))
