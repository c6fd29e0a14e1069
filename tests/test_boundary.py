"""The C-ABI boundary on CPU (no GPU): the library loads, exports every symbol include/mpo.h
declares, validates arguments with the documented status codes before touching the device, and
the product package never reaches the oracle."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpo.h")
PKG = os.path.join(ROOT, "paper_2309_12381_b200")


@pytest.fixture(scope="module")
def libs():
    from paper_2309_12381_b200 import _build, _lib
    _build.build()
    return _lib, _lib.load(False), _lib.load(True)


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpo_[a-z_0-9]+)\s*\(", src)))


def test_header_lists_the_north_star_entry_points():
    fns = header_functions()
    for f in ("mpo_split", "mpo_reconstruct", "mpo_sgd_step", "mpo_adam_step", "mpo_fused_backward_hook_step",
              "mpo_sharded_step"):
        assert f in fns


def test_every_declared_symbol_is_exported(libs):
    _lib, fma, exact = libs
    fns = header_functions()
    assert sorted(_lib.SYMBOLS) == fns
    for L in (fma, exact):
        for f in fns:
            assert hasattr(L, f), f


def test_build_flavours(libs):
    _lib, fma, exact = libs
    assert fma.mpo_build_exact() == 0
    assert exact.mpo_build_exact() == 1
    assert fma.mpo_norm_ws_doubles() >= 2


def test_sm100a_sass_present(libs):
    """The library carries sm_100a SASS (cuobjdump), not just PTX."""
    import subprocess
    from paper_2309_12381_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.lib_path(False)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _status(L, rc):
    return rc, L.mpo_last_error().decode()


def test_validation_errors(libs):
    _lib, L, _ = libs
    T, S, A = _lib.Tensor, _lib.SgdHP, _lib.AdamHP
    # bad value dtype
    rc, msg = _status(L, L.mpo_split(_lib.MPO_FP32, 16, 16, 16, 8, 0, 0, None))
    assert rc == _lib.MPO_EDTYPE and "value dtype" in msg
    # negative size
    rc, msg = _status(L, L.mpo_reconstruct(_lib.MPO_BF16, 16, 16, 16, -1, None))
    assert rc == _lib.MPO_EINVAL
    # misaligned pointer
    rc, msg = _status(L, L.mpo_split(_lib.MPO_FP16, 16, 18, 32, 8, 0, 0, None))
    assert rc == _lib.MPO_EALIGN
    # n == 0 is a no-op (OK) even with NULL pointers
    assert L.mpo_split(_lib.MPO_FP16, None, None, None, 0, 0, 0, None) == _lib.MPO_OK
    # table errors name the offending index
    tab = (T * 2)()
    for i in range(2):
        tab[i].value, tab[i].resid, tab[i].grad, tab[i].m, tab[i].v, tab[i].n = 16, 32, 48, 64, 80, 8
    tab[1].resid = 34
    hp = A(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0)
    rc, msg = _status(L, L.mpo_adam_step(_lib.MPO_BF16, _lib.MPO_BF16, tab, 2, C.byref(hp), 1, None, None))
    assert rc == _lib.MPO_EALIGN and "tensor 1" in msg
    tab[1].resid = 32
    tab[1].hp = 3
    rc, msg = _status(L, L.mpo_adam_step(_lib.MPO_BF16, _lib.MPO_BF16, tab, 2, C.byref(hp), 1, None, None))
    assert rc == _lib.MPO_EINVAL and "tensor 1" in msg
    tab[1].hp = 0
    # non-finite hyper-parameters rejected
    bad = A(float("nan"), 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0)
    rc, msg = _status(L, L.mpo_adam_step(_lib.MPO_BF16, _lib.MPO_BF16, tab, 2, C.byref(bad), 1, None, None))
    assert rc == _lib.MPO_EINVAL and "non-finite" in msg
    # step must be >= 1
    bad = A(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 0, 0)
    assert L.mpo_adam_step(_lib.MPO_BF16, _lib.MPO_BF16, tab, 2, C.byref(bad), 1, None, None) == _lib.MPO_EINVAL
    # unsupported grad dtype
    rc, _ = _status(L, L.mpo_adam_step(_lib.MPO_BF16, 7, tab, 2, C.byref(hp), 1, None, None))
    assert rc == _lib.MPO_EDTYPE
    # clipping without a workspace
    clip = A(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 1.0, 1, 0, 1, 0)
    assert L.mpo_adam_step(_lib.MPO_BF16, _lib.MPO_BF16, tab, 2, C.byref(clip), 1, None, None) == _lib.MPO_EINVAL
    # group count out of range
    assert L.mpo_adam_step(_lib.MPO_BF16, _lib.MPO_BF16, tab, 2, C.byref(hp), 0, None, None) == _lib.MPO_EINVAL
    # SGD: nesterov without momentum
    s = S(0.1, 0.0, 0.0, 0.0, 1.0, 1, 0, 0)
    rc, msg = _status(L, L.mpo_sgd_step(_lib.MPO_FP16, _lib.MPO_FP16, tab, 2, C.byref(s), 1, None, None))
    assert rc == _lib.MPO_EINVAL and "nesterov" in msg


def test_hook_refuses_global_clipping(libs):
    """P:93 / P:186: global operations are impossible inside the fused backward."""
    _lib, L, _ = libs
    one = _lib.Tensor(16, 32, 48, 64, 80, 8, 0, 0)
    clip = _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 1.0, 1, 0, 1, 0)
    rc, msg = _status(L, L.mpo_fused_backward_hook_step(_lib.MPO_ADAM, _lib.MPO_BF16, _lib.MPO_BF16, C.byref(one),
                                                        C.byref(clip), None, None))
    assert rc == _lib.MPO_EINVAL and "P:186" in msg
    assert L.mpo_fused_backward_hook_step(9, _lib.MPO_BF16, _lib.MPO_BF16, C.byref(one), C.byref(clip),
                                          None, None) == _lib.MPO_EINVAL
    # the found-inf skip needs a workspace; clip_value and max_grad_norm are exclusive
    skip = _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0, 0.0, 1, 0)
    rc, msg = _status(L, L.mpo_fused_backward_hook_step(_lib.MPO_ADAM, _lib.MPO_BF16, _lib.MPO_BF16, C.byref(one),
                                                        C.byref(skip), None, None))
    assert rc == _lib.MPO_EINVAL and "workspace" in msg
    both = _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 1.0, 1, 0, 1, 0, 0.5, 0, 0)
    tab = (_lib.Tensor * 1)(one)
    rc, msg = _status(L, L.mpo_adam_step(_lib.MPO_BF16, _lib.MPO_BF16, tab, 1, C.byref(both), 1, None, None))
    assert rc == _lib.MPO_EINVAL and "exclusive" in msg


def test_sharded_validation(libs):
    _lib, L, _ = libs
    hp = _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0)
    args = lambda comm, rank, world, n: (_lib.MPO_ADAM, comm, rank, world, _lib.MPO_BF16, 16, 32, 48, 64, 80, n,
                                         C.byref(hp), None, None)
    assert L.mpo_sharded_step(*args(0, 0, 2, 32)) == _lib.MPO_EINVAL          # NULL comm
    assert L.mpo_sharded_step(*args(1, 2, 2, 32)) == _lib.MPO_EINVAL          # rank >= world
    rc, msg = _status(L, L.mpo_sharded_step(*args(1, 0, 2, 24)))             # 24 not a multiple of 16
    assert rc == _lib.MPO_EINVAL and "8*world" in msg
    assert L.mpo_sharded_step(*args(1, 0, 2, 0)) == _lib.MPO_OK               # empty


def test_product_never_touches_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use oracle/."""
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b", src.replace("CPU oracle", "").replace("the oracle", "")), f
    assert "oracle" not in open(HEADER).read().replace("CPU oracle", "")


def test_python_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2309_12381_b200 import _build, _lib
    monkeypatch.setattr(_build, "lib_path", lambda exact=False: str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_libs", {})
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load(False)


def test_cpu_tensors_are_rejected():
    import torch
    from paper_2309_12381_b200 import MpoError, mpo_split
    with pytest.raises(MpoError, match="CUDA"):
        mpo_split(torch.zeros(8), torch.bfloat16, value=torch.zeros(8, dtype=torch.bfloat16),
                  resid=torch.zeros(8, dtype=torch.int16))


def test_grouped_sharded_and_sumsq_validation(libs):
    """mpo_sharded_step_grouped's segment table, mpo_grad_sumsq and mpo_comm_check validate their
    arguments before touching the device or the communicator (no GPU needed)."""
    _lib, L, _ = libs
    hp = (_lib.AdamHP * 2)(_lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0),
                           _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.1, 1.0, 0.0, 1, 0, 1, 0))

    def grouped(segs, nhp=2, n=64, world=2, vdt=_lib.MPO_BF16):
        arr = (_lib.Segment * len(segs))(*[_lib.Segment(*s) for s in segs])
        return _status(L, L.mpo_sharded_step_grouped(_lib.MPO_ADAM, 1, 0, world, vdt, 16, 32, 48, 64, 80, n, arr,
                                                      len(segs), C.cast(hp, C.c_void_p), nhp, None, None))
    rc, msg = grouped([(8, 0, 0)])
    assert rc == _lib.MPO_EINVAL and "segment 0" in msg                  # must start at 0
    rc, msg = grouped([(0, 0, 0), (4, 1, 1)])
    assert rc == _lib.MPO_EINVAL and "multiple of 8" in msg              # 16-B alignment of the pieces
    rc, msg = grouped([(0, 0, 0), (8, 1, 1)], vdt=49)                    # MPO_BF16_X8: int8 residuals
    assert rc == _lib.MPO_EINVAL and "multiple of 16" in msg
    rc, msg = grouped([(0, 0, 0), (32, 1, 1)])
    assert rc == _lib.MPO_EINVAL and "segment 1" in msg                  # beyond the 32-element shard
    rc, msg = grouped([(0, 2, 0)])
    assert rc == _lib.MPO_EINVAL and "group index" in msg
    rc, msg = grouped([(0, 0, 0)], nhp=17)
    assert rc == _lib.MPO_EINVAL
    # mpo_grad_sumsq
    tab = (_lib.Tensor * 1)(_lib.Tensor(0, 0, 48, 0, 0, 8, 0, 0))
    gs = (C.c_double * 1)(1.0)
    assert L.mpo_grad_sumsq(9, tab, 1, gs, 1, 16, 0, None) == _lib.MPO_EDTYPE
    assert L.mpo_grad_sumsq(_lib.MPO_BF16, tab, 1, gs, 1, None, 0, None) == _lib.MPO_EINVAL
    tab[0].grad = 50
    rc, msg = _status(L, L.mpo_grad_sumsq(_lib.MPO_BF16, tab, 1, gs, 1, 16, 0, None))
    assert rc == _lib.MPO_EALIGN and "tensor 0" in msg
    nan = (C.c_double * 1)(float("nan"))
    assert L.mpo_grad_sumsq(_lib.MPO_BF16, tab, 1, nan, 1, 16, 0, None) == _lib.MPO_EINVAL
    # communicator check: NULL refused (a live communicator is exercised by the GPU tests)
    assert L.mpo_comm_check(0) == _lib.MPO_EINVAL
    # norm_ready is for multi-tensor calls only
    one = _lib.Tensor(16, 32, 48, 64, 80, 8, 0, 0)
    ready = _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0, 0.0, 0, 1)
    rc, msg = _status(L, L.mpo_fused_backward_hook_step(_lib.MPO_ADAM, _lib.MPO_BF16, _lib.MPO_BF16, C.byref(one),
                                                        C.byref(ready), None, None))
    assert rc == _lib.MPO_EINVAL and "norm_ready" in msg


def test_graphed_step_validation(libs):
    """mpo_hp_block_fill / mpo_step_graphed validate before touching the device (no GPU needed)."""
    _lib, L, _ = libs
    assert L.mpo_hp_block_bytes(_lib.MPO_ADAM) > L.mpo_hp_block_bytes(_lib.MPO_SGD) > 16
    hp = _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0)
    buf = (C.c_uint8 * L.mpo_hp_block_bytes(_lib.MPO_ADAM))()
    assert L.mpo_hp_block_fill(_lib.MPO_ADAM, C.byref(hp), 1, 7, buf) == _lib.MPO_OK
    assert bytes(buf[-16:-8]) == (7).to_bytes(8, "little")        # the sequence number slot
    assert L.mpo_hp_block_fill(_lib.MPO_ADAM, C.byref(hp), 0, 7, buf) == _lib.MPO_EINVAL
    assert L.mpo_hp_block_fill(9, C.byref(hp), 1, 7, buf) == _lib.MPO_EINVAL
    bad = _lib.AdamHP(float("inf"), 0.9, 0.999, 1e-8, 0.0, 1.0, 0.0, 1, 0, 1, 0)
    assert L.mpo_hp_block_fill(_lib.MPO_ADAM, C.byref(bad), 1, 7, buf) == _lib.MPO_EINVAL
    tab = (_lib.Tensor * 1)(_lib.Tensor(16, 32, 48, 64, 80, 8, 0, 0))
    rc, msg = _status(L, L.mpo_step_graphed(_lib.MPO_ADAM, _lib.MPO_BF16, _lib.MPO_BF16, tab, 1, C.byref(hp), 1, None,
                                            4096, None, None, None))
    assert rc == _lib.MPO_EINVAL and "block" in msg
    rc, msg = _status(L, L.mpo_step_graphed(_lib.MPO_ADAM, _lib.MPO_BF16, _lib.MPO_BF16, tab, 1, C.byref(hp), 1, buf,
                                            4100, None, None, None))
    assert rc == _lib.MPO_EALIGN


def _res_usage(path):
    import re
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-res-usage", path], capture_output=True, text=True).stdout
    res = {}
    name = None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        if name and "REG:" in line:
            res[name] = {k: int(v) for k, v in re.findall(r"(REG|STACK|LOCAL|SHARED):(\d+)", line)}
            name = None
    return res


@pytest.mark.parametrize("exact", [True, False])
def test_kernel_resources(exact):
    """Build-artifact guard (cuobjdump, no GPU): no kernel spills to local memory, and the
    per-thread-load step kernel keeps two CTAs of 256 threads per SM (<= 128 registers) in all
    but a handful of instantiations -- a runtime select of two hyper-parameter banks once pushed
    60 of them to 160 registers."""
    from paper_2309_12381_b200 import _build
    path = _build.lib_path(exact)
    if not os.path.exists(path):
        pytest.skip("library not built")
    res = _res_usage(path)
    assert len(res) > 300, len(res)
    assert not [k for k, v in res.items() if v.get("LOCAL", 0) > 0]
    lsu = {k: v for k, v in res.items() if k.startswith("_ZN3mpo11step_kernel")}
    assert len(lsu) >= 144
    high = [k for k, v in lsu.items() if v["REG"] > 128]
    assert len(high) <= 8, (len(high), high[:4])
