"""Host-side logic of the Python binding (no GPU): storage-format codes, residual containers,
per-step seeds, argument rejection before any device work."""
import pytest
import torch

import paper_2309_12381_b200 as mpo
from paper_2309_12381_b200 import api
from paper_2309_12381_b200._lib import MPO_BF16, MPO_FP16, MpoError


def test_format_codes_match_the_header():
    assert api.format_code(torch.float16, "rne") == MPO_FP16 == 0
    assert api.format_code(torch.bfloat16, "rne") == MPO_BF16 == 1
    assert api.format_code(torch.float16, "rtz") == 16 and api.format_code(torch.bfloat16, "rtz") == 17
    assert api.format_code(torch.float16, "sr") == 32
    assert api.format_code(torch.float16, "x8") == 48 and api.format_code(torch.bfloat16, "x8") == 49
    assert api.format_code(torch.float16, "x8z") == 64 and api.format_code(torch.bfloat16, "x8z") == 65
    header = open(__import__("os").path.join(__import__("os").path.dirname(__file__), "..", "include", "mpo.h")).read()
    for name, code in (("MPO_FP16_RTZ", 16), ("MPO_BF16_RTZ", 17), ("MPO_FP16_SR", 32), ("MPO_FP16_X8", 48),
                       ("MPO_BF16_X8", 49), ("MPO_FP16_X8Z", 64), ("MPO_BF16_X8Z", 65)):
        assert f"{name} = {code}" in header


def test_format_errors():
    with pytest.raises(MpoError, match="fp16"):
        api.format_code(torch.bfloat16, "sr")          # SR is defined for fp16 only
    with pytest.raises(MpoError, match="scheme"):
        api.format_code(torch.float16, "nope")
    with pytest.raises(MpoError):
        api.format_code(torch.float32, "rne")


def test_resid_containers_and_seeds():
    assert api.resid_dtype("rne") == api.resid_dtype("rtz") == api.resid_dtype("sr") == torch.int16
    assert api.resid_dtype("x8") == torch.int8 and api.resid_dtype("x8z") == torch.uint8
    seeds = {api.step_seed(7, t) for t in range(1000)}
    assert len(seeds) == 1000 and all(0 <= s < 2 ** 64 for s in seeds)
    assert api.step_seed(7, 3) != api.step_seed(8, 3)


def test_hp_structs_marshal_all_fields():
    a = mpo.AdamParams(lr=1e-3, beta1=0.8, beta2=0.95, eps=1e-6, weight_decay=0.1, grad_scale=0.5, max_grad_norm=2.0,
                       adamw=False, step=7, seed=9, clip_value=0.0, skip_nonfinite=True).c()
    assert (a.lr, a.beta1, a.beta2, a.eps, a.weight_decay, a.grad_scale, a.max_grad_norm) == \
        (1e-3, 0.8, 0.95, 1e-6, 0.1, 0.5, 2.0)
    assert (a.adamw, a.step, a.seed, a.skip_nonfinite) == (0, 7, 9, 1)
    s = mpo.SgdParams(lr=0.1, momentum=0.9, dampening=0.1, weight_decay=1e-4, nesterov=False, first_step=True,
                      seed=3, clip_value=0.5).c()
    assert (s.lr, s.momentum, s.dampening, s.weight_decay, s.first_step, s.seed, s.clip_value) == \
        (0.1, 0.9, 0.1, 1e-4, 1, 3, 0.5)


def test_table_rejects_bad_columns_before_device_work():
    v = torch.zeros(8, dtype=torch.bfloat16)
    with pytest.raises(MpoError, match="CUDA"):
        api.TensorTable([v], [torch.zeros(8, dtype=torch.int16)], [v], [torch.zeros(8)], [torch.zeros(8)])
    with pytest.raises(MpoError, match="resid"):
        api.TensorTable([v], [torch.zeros(8, dtype=torch.int8)], [v], [None], [None])
    with pytest.raises(MpoError, match="length"):
        api.TensorTable([v], [], [v], [None], [None])


def test_optimizer_refuses_cpu_parameters():
    with pytest.raises(MpoError, match="CUDA"):
        mpo.ResidualAdamW([torch.nn.Parameter(torch.zeros(4))], fmt=torch.bfloat16)
