"""User-facing optimizers: residual-compensated SGD-momentum and Adam/AdamW on a 16-bit model.

``ResidualSGD`` / ``ResidualAdamW`` hold, per parameter, the int16 residual and the fp32 state
("Extra bits are stored by the optimizer and do not require any modification in the training
framework").  The parameter tensor itself is the 16-bit value.  Two ways to step:

* ``step()``: one multi-tensor launch over all parameters with a gradient ("one only
  stream of values"); global-norm clipping available (``max_grad_norm``);
* ``install_backward_hooks()``: the step runs inside backward from each parameter's
  post-accumulate-grad hook and the gradient is freed immediately; global operations
  are refused there.

Everything numeric runs in libmpo (api.py marshals arguments only).
"""
from __future__ import annotations

import ctypes as C
import weakref
from typing import Iterable, Optional

import torch

from . import api
from ._lib import MPO_ADAM, MPO_SGD, MPO_MAX_HP_GROUPS, MpoError, Tensor

_16 = (torch.float16, torch.bfloat16)


def _weak_hook(opt):
    """A post-accumulate-grad hook that refers to its optimizer weakly: the tensor's hook table is
    held from C++, where Python's cycle collector cannot see it, so a strong reference would keep
    the optimizer and its state alive forever."""
    ref = weakref.ref(opt)

    def hook(p):
        o = ref()
        if o is not None:
            o._hook(p)
    return hook


class _ResidualOptimizer(torch.optim.Optimizer):
    _kind = None

    def __init__(self, params, defaults, fmt: Optional[torch.dtype], exact: bool, scheme: str = "rne",
                 seed: int = 0, clip_value: float = 0.0, skip_nonfinite: bool = False):
        super().__init__(params, defaults)
        self.exact = exact
        self.scheme = scheme
        self.seed = int(seed)
        self.clip_value = float(clip_value or 0.0)
        self.skip_nonfinite = bool(skip_nonfinite)
        self._hooks = []
        self._tables = {}
        self._norm_ws = None
        idx = 0
        for group in self.param_groups:
            for p in group["params"]:
                self._init_param(p, fmt, idx)
                idx += 1

    # -- state ------------------------------------------------------------------------------
    def _init_param(self, p: torch.Tensor, fmt, idx: int):
        if not p.is_cuda:
            raise MpoError(1, "parameters must live on a CUDA device (no CPU path)")
        st = self.state[p]
        st["index"] = idx            # also the stochastic-rounding stream of this parameter
        if p.dtype == torch.float32:
            if fmt not in _16:
                raise MpoError(3, "an fp32 parameter needs fmt=torch.float16 or torch.bfloat16 to be split")
            with torch.no_grad():
                value, resid = api.mpo_split(p.data.contiguous(), fmt, exact=self.exact, scheme=self.scheme,
                                             seed=api.step_seed(self.seed, 0), sr_stream=idx)
                p.data = value
            st["resid"] = resid
        elif p.dtype in _16:
            # a 16-bit value is exactly representable: its residual is 0 under every scheme (P1)
            api.format_code(p.dtype, self.scheme)
            st["resid"] = torch.zeros(p.shape, dtype=api.resid_dtype(self.scheme), device=p.device)
        else:
            raise MpoError(3, f"unsupported parameter dtype {p.dtype}")
        st["step"] = 0
        self._init_state(p, st)

    def _init_state(self, p, st):
        raise NotImplementedError

    def fp32_params(self):
        """The full-precision weights, reconstructed from value + residual."""
        out = []
        for group in self.param_groups:
            for p in group["params"]:
                out.append(api.mpo_reconstruct(p.data, self.state[p]["resid"], exact=self.exact,
                                               scheme=self.scheme))
        return out

    # -- multi-tensor step -----------------------------------------------------------------
    def _table_for(self, params):
        key = tuple(id(p) for p in params)
        tab = self._tables.get(key)
        grads = [p.grad for p in params]
        if tab is None:
            gi = {id(p): gi for gi, g in enumerate(self.param_groups) for p in g["params"]}
            st = [self.state[p] for p in params]
            tab = api.TensorTable([p.data for p in params], [s["resid"] for s in st], grads,
                                  [s.get("m") for s in st], [s.get("v") for s in st],
                                  [0] * len(params), scheme=self.scheme, sr_streams=[s["index"] for s in st])
            tab._group_of = [gi[id(p)] for p in params]
            self._tables[key] = tab
        elif [g.data_ptr() for g in grads] != tab.grad_ptrs:
            tab.set_grads(grads)
        return tab

    @torch.no_grad()
    def step(self, closure=None):
        if closure is not None:
            raise MpoError(1, "closure optimizers are not supported (the step is fused, P:194)")
        params = [p for g in self.param_groups for p in g["params"] if p.grad is not None]
        if not params:
            return None
        by_dtype = {}
        for p in params:
            by_dtype.setdefault((p.dtype, p.grad.dtype), []).append(p)
        for plist in by_dtype.values():
            tab = self._table_for(plist)
            # hyper-parameter groups: one per (param group, step)
            keys, hp_index = {}, []
            for p, gi in zip(plist, tab._group_of):
                self.state[p]["step"] += 1
                k = (gi, self.state[p]["step"])
                hp_index.append(keys.setdefault(k, len(keys)))
            if len(keys) > MPO_MAX_HP_GROUPS:
                raise MpoError(1, "more than 16 distinct (group, step) pairs in one step")
            for i, h in enumerate(hp_index):
                tab.arr[i].hp = h
            hps = [self._hp(self.param_groups[gi], stp) for (gi, stp) in keys]
            self._launch(tab, hps)
        return None

    # -- hook mode ---------------------------------------------------------------------------
    def install_backward_hooks(self, batch_below: int = 1 << 16, flush_elems: int = 1 << 22):
        """Step each parameter inside backward, as soon as its gradient is accumulated, then free
        the gradient.  Returns the hook handles.

        Parameters smaller than ``batch_below`` elements (biases, norms) are not launched one by
        one: their gradients are held until ``flush_elems`` elements are pending or the backward
        ends, then stepped by one multi-tensor launch (bounded transient memory, far fewer
        launches).  ``batch_below=0`` steps every parameter individually; batching is off with
        ``skip_nonfinite`` (whose hook-mode skip is per parameter).  The hooks hold the optimizer
        weakly: keep a reference to it for as long as training runs."""
        self._check_hook_mode()
        self._batch_below = 0 if self.skip_nonfinite else int(batch_below)
        self._flush_elems = int(flush_elems)
        self._pending = []
        self._pending_elems = 0
        self._flush_queued = False
        self._hp_c, self._codes = {}, {}
        for gi, group in enumerate(self.param_groups):
            for p in group["params"]:
                st = self.state[p]
                row = Tensor()
                row.value = p.data.data_ptr()
                row.resid = st["resid"].data_ptr()
                row.m = st["m"].data_ptr() if st.get("m") is not None else None
                row.v = st["v"].data_ptr() if st.get("v") is not None else None
                row.n = p.numel()
                row.sr_stream = st["index"]
                st["row"] = row
                st["group"] = gi
                self._hooks.append(p.register_post_accumulate_grad_hook(_weak_hook(self)))
        return list(self._hooks)

    def remove_backward_hooks(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []

    def _hook(self, p: torch.Tensor):
        st = self.state[p]
        g = p.grad
        st["step"] += 1
        if p.numel() < self._batch_below:
            self._pending.append((p, g))
            self._pending_elems += p.numel()
            p.grad = None            # the pending list keeps the (small) gradient until the flush
            if not self._flush_queued:
                torch.autograd.Variable._execution_engine.queue_callback(self._flush_pending)
                self._flush_queued = True
            if self._pending_elems >= self._flush_elems:
                self._flush_pending(final=False)
            return
        row = st["row"]
        row.grad = g.data_ptr()
        # host cost per hook matters when backward is short: the ctypes hyper-parameters are built
        # once per (group, step) and shared by the group's parameters; format codes are cached
        key = (st["group"], st["step"])
        hp = self._hp_c.get(key)
        if hp is None:
            if len(self._hp_c) > 64:
                self._hp_c.clear()
            hp = self._hp_c[key] = self._hp(self.param_groups[st["group"]], st["step"]).c()
        codes = self._codes.get((p.dtype, g.dtype))
        if codes is None:
            codes = self._codes[(p.dtype, g.dtype)] = (api.format_code(p.dtype, self.scheme), api.dtype_code(g.dtype))
        api.mpo_fused_backward_hook_step(self._kind, codes[0], codes[1], row, hp, exact=self.exact,
                                         norm_ws=self._ws(p.device) if self.skip_nonfinite else None)
        p.grad = None   # freed now; stream order makes the block's reuse safe

    def _flush_pending(self, final: bool = True):
        """One multi-tensor launch over the batched small parameters of this backward."""
        if final:
            self._flush_queued = False
        if not self._pending:
            return
        pending, self._pending, self._pending_elems = self._pending, [], 0
        with torch.no_grad():
            by_dtype = {}
            for p, g in pending:
                by_dtype.setdefault((p.dtype, g.dtype), []).append((p, g))
            for items in by_dtype.values():
                ps = [p for p, _ in items]
                sts = [self.state[p] for p in ps]
                keys, hp_index = {}, []
                for s_ in sts:
                    hp_index.append(keys.setdefault((s_["group"], s_["step"]), len(keys)))
                tab = api.TensorTable([p.data for p in ps], [s_["resid"] for s_ in sts], [g for _, g in items],
                                      [s_.get("m") for s_ in sts], [s_.get("v") for s_ in sts], hp_index,
                                      scheme=self.scheme, sr_streams=[s_["index"] for s_ in sts])
                hps = [self._hp(self.param_groups[gi], stp) for (gi, stp) in keys]
                if len(hps) > MPO_MAX_HP_GROUPS:
                    raise MpoError(1, "more than 16 distinct (group, step) pairs in one flush")
                self._launch(tab, hps)
        del pending              # the gradients are released (stream order keeps reuse safe)

    # -- loss scaling: found-inf -------------------------------------------------------------
    def _ws(self, device):
        if self._norm_ws is None:
            self._norm_ws = torch.zeros(api.norm_ws_doubles(self.exact), dtype=torch.float64, device=device)
        return self._norm_ws

    def found_inf(self, reset: bool = True) -> bool:
        """skip_nonfinite: whether a non-finite scaled gradient was seen -- by the last step() (which
        then updated nothing), or by any hook of the backward passes since the last reset (hook
        mode skips only the offending parameters).  Synchronises with the device."""
        if self._norm_ws is None:
            return False
        ws = self._norm_ws
        bad = not bool(torch.isfinite(ws[0]).item()) or not bool(torch.isfinite(ws[-1]).item())
        if reset:
            ws[0] = 0.0
            ws[-1] = 0.0
        return bad

    def _check_hook_mode(self):
        pass

    def _hp(self, group, step):
        raise NotImplementedError

    def _launch(self, tab, hps):
        raise NotImplementedError


class ResidualSGD(_ResidualOptimizer):
    """SGD(-momentum) on 16-bit parameters with residual-compensated updates (torch.optim.SGD
    semantics, R6)."""
    _kind = MPO_SGD

    def __init__(self, params: Iterable, lr: float, momentum: float = 0.0, dampening: float = 0.0,
                 weight_decay: float = 0.0, nesterov: bool = False, grad_scale: float = 1.0,
                 fmt: Optional[torch.dtype] = None, exact: bool = False, scheme: str = "rne", seed: int = 0,
                 clip_value: float = 0.0, skip_nonfinite: bool = False):
        defaults = dict(lr=lr, momentum=momentum, dampening=dampening, weight_decay=weight_decay,
                        nesterov=nesterov, grad_scale=grad_scale)
        super().__init__(params, defaults, fmt, exact, scheme, seed, clip_value, skip_nonfinite)

    def _init_state(self, p, st):
        group = next(g for g in self.param_groups if any(q is p for q in g["params"]))  # noqa
        st["m"] = torch.zeros(p.shape, dtype=torch.float32, device=p.device) if group["momentum"] != 0 else None
        st["v"] = None

    def _hp(self, g, step):
        return api.SgdParams(lr=g["lr"], momentum=g["momentum"], dampening=g["dampening"],
                             weight_decay=g["weight_decay"], grad_scale=g["grad_scale"], nesterov=g["nesterov"],
                             first_step=(step == 1), seed=api.step_seed(self.seed, step),
                             clip_value=self.clip_value, skip_nonfinite=self.skip_nonfinite)

    def _launch(self, tab, hps):
        ws = self._ws(tab.values[0].device) if self.skip_nonfinite else None
        api.mpo_sgd_step(tab, hps, norm_ws=ws, exact=self.exact)


class ResidualAdamW(_ResidualOptimizer):
    """Adam / AdamW on 16-bit parameters with residual-compensated updates (torch.optim.Adam
    semantics, R6).  ``max_grad_norm`` enables global-norm clipping in ``step()``."""
    _kind = MPO_ADAM

    def __init__(self, params: Iterable, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, adamw: bool = True, grad_scale: float = 1.0,
                 max_grad_norm: Optional[float] = None, fmt: Optional[torch.dtype] = None, exact: bool = False,
                 scheme: str = "rne", seed: int = 0, clip_value: float = 0.0, skip_nonfinite: bool = False):
        defaults = dict(lr=lr, betas=tuple(betas), eps=eps, weight_decay=weight_decay, adamw=adamw,
                        grad_scale=grad_scale)
        self.max_grad_norm = float(max_grad_norm) if max_grad_norm else 0.0
        super().__init__(params, defaults, fmt, exact, scheme, seed, clip_value, skip_nonfinite)

    def _init_state(self, p, st):
        st["m"] = torch.zeros(p.shape, dtype=torch.float32, device=p.device)
        st["v"] = torch.zeros(p.shape, dtype=torch.float32, device=p.device)

    def _check_hook_mode(self):
        if self.max_grad_norm > 0:
            raise MpoError(1, "global-norm clipping needs every gradient at once: impossible in the fused "
                              "backward (P:93, P:186); use step() instead")

    def _hp(self, g, step):
        b1, b2 = g["betas"]
        return api.AdamParams(lr=g["lr"], beta1=b1, beta2=b2, eps=g["eps"], weight_decay=g["weight_decay"],
                              grad_scale=g["grad_scale"], max_grad_norm=self.max_grad_norm, adamw=g["adamw"],
                              step=step, seed=api.step_seed(self.seed, step), clip_value=self.clip_value,
                              skip_nonfinite=self.skip_nonfinite)

    def _launch(self, tab, hps):
        ws = self._ws(tab.values[0].device) if (self.max_grad_norm > 0 or self.skip_nonfinite) else None
        api.mpo_adam_step(tab, hps, norm_ws=ws, exact=self.exact)

    def last_grad_sumsq(self) -> Optional[torch.Tensor]:
        """Device scalar: the fp64 sum of squares of the scaled gradients of the last clipped step."""
        return None if self._norm_ws is None else self._norm_ws[0]
