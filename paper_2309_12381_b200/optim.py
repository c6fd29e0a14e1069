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
import math
import time
import weakref
from typing import Iterable, Optional

import numpy as np
import torch

from . import api
from ._lib import MPO_ADAM, MPO_SGD, MPO_MAX_HP_GROUPS, MpoError, Tensor

_16 = (torch.float16, torch.bfloat16)


class _GroupDict(dict):
    """A param group that pushes hyper-parameter changes (e.g. an LR scheduler's
    ``group["lr"] = ...``) to the native hooks, which build each call's struct without Python."""

    def __init__(self, d, on_change):
        super().__init__(d)
        self._on_change = on_change

    def __setitem__(self, k, v):
        super().__setitem__(k, v)
        self._on_change()

    def update(self, *a, **kw):
        super().update(*a, **kw)
        self._on_change()


def _native_finalize(ns, mod, params):
    """The optimizer is gone: disarm the native state (its hooks then do nothing) and take the
    hooks off the parameters that are still alive."""
    ns.disarm()
    for ref in params:
        p = ref()
        if p is not None:
            try:
                mod.uninstall(p)
            except Exception:
                pass


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
    # torch.amp.GradScaler.step() protocol: it sets `self.grad_scale` (the loss scale, a device
    # tensor) and `self.found_inf` (device tensor, nonzero when a scaled gradient was not finite)
    # before calling step(), which then unscales inside the fused step and skips a non-finite one
    _step_supports_amp_scaling = True
    _amp_inv = 1.0

    def __init__(self, params, defaults, fmt: Optional[torch.dtype], exact: bool, scheme: str = "rne",
                 seed: int = 0, clip_value: float = 0.0, skip_nonfinite: bool = False):
        self._fmt = fmt
        super().__init__(params, defaults)
        self.exact = exact
        self.scheme = scheme
        self.seed = int(seed)
        self.clip_value = float(clip_value or 0.0)
        self.skip_nonfinite = bool(skip_nonfinite)
        self._hooks = []
        self._tables = {}
        self._norm_ws = None
        # hook mode: the ctypes table row and group of each parameter, kept OUT of self.state so
        # state_dict() stays plain tensors and ints (picklable)
        self._rows = {}
        # skip_nonfinite: the step counts a skipped update must not advance are rolled back once its
        # found-inf flag has reached the host (deferred, no synchronisation in step())
        self._skip_check = None
        self._hook_S = None
        self._native = None          # native (C++) hook state, see install_backward_hooks
        # per-parameter step counts, one int64 each: state[p]["step"] is a 0-dim view of this host
        # buffer, which the native hooks update in place (one source of truth for both paths)
        self._steps = torch.zeros(sum(len(g["params"]) for g in self.param_groups), dtype=torch.int64)
        self._steps_np = self._steps.numpy()     # the same memory: host-side updates without torch ops
        idx = 0
        for group in self.param_groups:
            for p in group["params"]:
                self._init_param(p, fmt, idx)
                idx += 1

    def add_param_group(self, param_group):
        """torch.optim semantics: a new group joins the optimizer (its fp32 parameters are split into
        16-bit value + residual like the constructor's, their step counts start at 0).  Not while
        the backward hooks or the graph-replayed step are installed (they hold the tables)."""
        if not hasattr(self, "_steps"):          # called by torch's constructor
            return super().add_param_group(param_group)
        if self._hooks or self._native is not None or getattr(self, "_graph", None) is not None:
            raise MpoError(1, "add_param_group: remove the backward hooks / graph step first")
        self._resolve_skips()
        self._pull_native_steps()
        super().add_param_group(param_group)
        new = self.param_groups[-1]["params"]
        n_old = self._steps.numel()
        steps = torch.zeros(n_old + len(new), dtype=torch.int64)
        steps[:n_old] = self._steps
        self._steps, self._steps_np = steps, steps.numpy()
        for group in self.param_groups[:-1]:
            for p in group["params"]:
                self.state[p]["step"] = self._steps[self.state[p]["index"]]
        for i, p in enumerate(new):
            self._init_param(p, self._fmt, n_old + i)
        self._tables.clear()

    # -- state ------------------------------------------------------------------------------
    def _init_param(self, p: torch.Tensor, fmt, idx: int):
        if not p.is_cuda:
            raise MpoError(1, "parameters must live on a CUDA device (no CPU path)")
        dev = self.param_groups[0]["params"][0].device
        if p.device != dev:
            # one launch covers a whole table on one device's stream: one optimizer per device
            raise MpoError(1, f"parameters on {p.device} and {dev}: use one optimizer per device")
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
        st["step"] = self._steps[idx]
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

    # -- checkpoint / resume ---------------------------------------------------------------
    def state_dict(self):
        """torch-style state dict: per parameter its residual (int16 / int8, the paper's extra bits,
        P:82 "Extra bits are stored by the optimizer"), fp32 m / v, the int step count and the
        stochastic-rounding stream index; plus the param groups and an "mpo" entry (storage scheme,
        seed, gradient surgery).  The 16-bit values themselves are the parameters (model.state_dict()).
        Tensors are referenced, not copied (torch.save serialises them)."""
        self._resolve_skips()
        self._pull_native_steps()
        sd = super().state_dict()
        sd["param_groups"] = [{k: v for k, v in g.items()} for g in sd["param_groups"]]
        sd["state"] = {k: {**st, "step": int(st["step"])} for k, st in sd["state"].items()}
        sd["mpo"] = {"format": 1, "kind": "adam" if self._kind == MPO_ADAM else "sgd", "scheme": self.scheme,
                     "seed": self.seed, "clip_value": self.clip_value, "skip_nonfinite": self.skip_nonfinite,
                     "max_grad_norm": getattr(self, "max_grad_norm", 0.0)}
        return sd

    def load_state_dict(self, state_dict):
        """Restore a state_dict() of the same parameter layout.  Unlike torch's base class (which
        casts floating state to the parameter's dtype), residual / m / v keep their own dtypes and
        are copied INTO the existing device buffers (shape and dtype checked), so the cached
        multi-tensor tables and hook rows stay valid; they are rebuilt anyway."""
        meta = state_dict.get("mpo")
        if meta is None:
            raise MpoError(1, "not a residual-optimizer state dict (no 'mpo' entry)")
        kind = "adam" if self._kind == MPO_ADAM else "sgd"
        if meta.get("kind") != kind or meta.get("scheme") != self.scheme:
            raise MpoError(3, f"state dict of a {meta.get('kind')}/{meta.get('scheme')} optimizer, this one is "
                              f"{kind}/{self.scheme}")
        saved = state_dict["param_groups"]
        if len(saved) != len(self.param_groups) or any(len(a["params"]) != len(b["params"])
                                                       for a, b in zip(saved, self.param_groups)):
            raise MpoError(1, "state dict has a different parameter group layout")
        self._resolve_skips()
        id_map = {old: p for a, b in zip(saved, self.param_groups) for old, p in zip(a["params"], b["params"])}
        with torch.no_grad():
            for k, st in state_dict["state"].items():
                p = id_map[k]
                cur = self.state[p]
                for key in ("resid", "m", "v"):
                    src, dst = st.get(key), cur.get(key)
                    if (src is None) != (dst is None):
                        raise MpoError(1, f"parameter {k}: '{key}' present in only one of state dict / optimizer")
                    if src is None:
                        continue
                    if src.dtype != dst.dtype or tuple(src.shape) != tuple(dst.shape):
                        raise MpoError(3, f"parameter {k}: '{key}' is {src.dtype}{tuple(src.shape)}, "
                                          f"expected {dst.dtype}{tuple(dst.shape)}")
                    dst.copy_(src)
                cur["step"].fill_(int(st["step"]))
                cur["index"] = int(st["index"])
        for g, a in zip(self.param_groups, saved):
            for key, val in a.items():
                if key != "params":
                    g[key] = val
        self.seed = int(meta["seed"])
        self.clip_value = float(meta["clip_value"])
        self.skip_nonfinite = bool(meta["skip_nonfinite"])
        if hasattr(self, "max_grad_norm"):
            self.max_grad_norm = float(meta.get("max_grad_norm", 0.0))
        self._tables.clear()
        if self._hooks:
            self._build_rows()
            self._hp_c = {}
        if self._native is not None:
            self._native.resolve()
            for gi in range(len(self.param_groups)):
                self._push_group(gi)

    # -- loss scaling: step counts of skipped updates (deferred) -----------------------------
    def _queue_skip_check(self, params, dev_S):
        """Queue a device->host copy of the step's S (non-blocking) to learn later whether the
        update was skipped; params' step counts are then rolled back (torch's GradScaler does not
        step the optimizer, so its bias corrections never count a skipped step)."""
        host = torch.empty(dev_S.numel(), dtype=torch.float64, pin_memory=True)
        host.copy_(dev_S, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._skip_check = (params, host, ev)

    def _resolve_skips(self):
        chk, self._skip_check = self._skip_check, None
        if chk is None:
            return
        params, host, ev = chk
        ev.synchronize()
        bad = [not math.isfinite(x) for x in host.tolist()]
        if len(bad) == 1:
            bad = bad * len(params)
        for p, b in zip(params, bad):
            if b:
                self._steps_np[self.state[p]["index"]] -= 1

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
            tab._idx = np.array([s["index"] for s in st], dtype=np.int64)
            self._tables[key] = tab
        elif [g.data_ptr() for g in grads] != tab.grad_ptrs:
            tab.set_grads(grads)
        return tab

    @torch.no_grad()
    def step(self, closure=None):
        if closure is not None:
            raise MpoError(1, "closure optimizers are not supported (the step is fused, P:194)")
        found_inf = self.__dict__.get("found_inf")
        if found_inf is not None:            # called by torch.amp.GradScaler.step()
            if self._hooks or self._native is not None or getattr(self, "_graph", None) is not None:
                raise MpoError(1, "GradScaler: the backward hooks / graph step update inside backward / the "
                                  "graph; use grad_scale= and skip_nonfinite= instead (P:193)")
            # the scaler's own inf check has run (it reads every gradient); one host read of the
            # flag and the scale, like torch's non-fused optimizer path
            if float(found_inf) != 0.0:
                return None                  # skipped: no update, no step count (R16)
            scale = self.__dict__.get("grad_scale")
            self._amp_inv = 1.0 / float(scale) if scale is not None else 1.0
            try:
                return self._step_eager()
            finally:
                self._amp_inv = 1.0
        if getattr(self, "_graph", None) is not None:
            return self._graph_step()        # prepare_step() did the host side
        return self._step_eager()

    def _step_eager(self):
        self._resolve_skips()
        params = [p for g in self.param_groups for p in g["params"] if p.grad is not None]
        if not params:
            return None
        self._pull_native_steps()            # a multi-tensor step between native-hook backwards
        by_dtype = {}
        for p in params:
            by_dtype.setdefault((p.dtype, p.grad.dtype), []).append(p)
        launches = []
        for plist in by_dtype.values():
            tab = self._table_for(plist)
            # hyper-parameter groups: one per (param group, step); the counts advance in the shared
            # host buffer with one vectorised numpy update (no per-parameter torch op)
            self._steps_np[tab._idx] += 1
            keys, hp_index = {}, []
            for gi, stp in zip(tab._group_of, self._steps_np[tab._idx].tolist()):
                hp_index.append(keys.setdefault((gi, stp), len(keys)))
            hps = [self._hp(self.param_groups[gi], stp) for (gi, stp) in keys]
            if len(keys) > MPO_MAX_HP_GROUPS:
                # more (group, step) pairs than one launch's hyper-parameter bank holds (e.g. layer-
                # wise lr decay): one launch per 16 of them, over the parameters that use them
                for c in range(0, len(keys), MPO_MAX_HP_GROUPS):
                    sel = [i for i, h in enumerate(hp_index) if c <= h < c + MPO_MAX_HP_GROUPS]
                    sub = self._table_for([plist[i] for i in sel])
                    for r, i in enumerate(sel):
                        sub.arr[r].hp = hp_index[i] - c
                    sub._hp_index = None
                    launches.append((sub, hps[c:c + MPO_MAX_HP_GROUPS]))
                continue
            if hp_index != getattr(tab, "_hp_index", None):     # usually unchanged from the last step
                for i, h in enumerate(hp_index):
                    tab.arr[i].hp = h
                tab._hp_index = hp_index
            launches.append((tab, hps))
        need_norm = self._needs_norm()
        if need_norm and len(launches) > 1:
            # one S over every table of the step (global-norm clipping is over ALL gradients, R9;
            # the found-inf skip is all-or-nothing): shared pre-pass, then norm_ready launches
            ws = self._ws(params[0].device)
            for i, (tab, hps) in enumerate(launches):
                api.mpo_grad_sumsq(tab, [h.grad_scale for h in hps], ws, accumulate=i > 0, exact=self.exact)
                for h in hps:
                    h.norm_ready = True
        for tab, hps in launches:
            self._launch(tab, hps)
        if self.skip_nonfinite:
            self._queue_skip_check(params, self._ws(params[0].device)[:1])
        return None

    def _needs_norm(self):
        return self.skip_nonfinite or getattr(self, "max_grad_norm", 0.0) > 0

    # -- CUDA-graph step -------------------------------------------------------------------
    def enable_graph_step(self):
        """Make step() capturable ONCE in a CUDA graph together with the rest of the training
        iteration, then replayed every step (mpo_step_graphed: the step's hyper-parameters are not
        kernel arguments but a block copied from pinned host memory at execution time)::

            opt.enable_graph_step()
            # warm up eagerly so every parameter has its gradient buffer (fixed addresses)
            with torch.cuda.graph(g):
                loss = model(x).loss; loss.backward(); opt.step()     # captures, runs nothing
            for it in range(...):
                opt.prepare_step()          # step counts + this step's lr / bias corrections
                g.replay()

        (Eagerly, ``opt.prepare_step(); opt.step()`` is one ordinary step.)  prepare_step() first
        waits until the previous step's hyper-parameter copy has happened (the device echoes each
        block's sequence number to a pinned word right after its copy) or the current stream is
        idle, so it never rewrites a block a pending replay still has to read.  Bit-identical to
        the eager step() sequence.  Not with the backward hooks or skip_nonfinite (whose step-count
        rollback reads back from the device)."""
        if self.skip_nonfinite:
            raise MpoError(1, "graph step: skip_nonfinite needs a device read-back per step")
        if self._hooks or self._native is not None:
            raise MpoError(1, "graph step: not with the backward hooks (they step inside backward)")
        self._graph = {}
        self._graph_seq = 0

    def prepare_step(self):
        """Host side of a graph-replayed step (see enable_graph_step): advance the step counts and
        write this step's hyper-parameters into the pinned blocks the captured copies read."""
        if getattr(self, "_graph", None) is None:
            raise MpoError(1, "call enable_graph_step() first")
        # never rewrite a block an issued step still has to copy: wait until the device echoed the
        # last sequence number -- or the stream ran dry (a block prepared but never replayed will
        # not be copied any more)
        stream = torch.cuda.current_stream()
        for ent in self._graph.values():
            while int(ent["ack"][0]) != self._graph_seq and not stream.query():
                time.sleep(0)
        self._graph_seq += 1
        self._graph_tables(advance=True)

    def _graph_tables(self, advance):
        params = [p for g in self.param_groups for p in g["params"] if p.grad is not None]
        by_dtype = {}
        for p in params:
            by_dtype.setdefault((p.dtype, p.grad.dtype), []).append(p)
        if self._needs_norm() and len(by_dtype) > 1:
            # each graphed launch runs its own norm pre-pass: one global S over tables of different
            # gradient dtypes would need the eager step's shared pre-pass
            raise MpoError(1, "graph step: global-norm clipping over gradients of different dtypes")
        if len(self.param_groups) > MPO_MAX_HP_GROUPS:
            raise MpoError(1, f"graph step: at most {MPO_MAX_HP_GROUPS} param groups (one hyper-parameter bank)")
        for key, plist in by_dtype.items():
            tab = self._table_for(plist)
            ent = self._graph.get(key)
            if ent is not None and ent["tab"] is not tab:
                raise MpoError(1, "graph step: the gradients moved since capture (keep them allocated)")
            if advance:
                self._steps_np[tab._idx] += 1
            groups = sorted(set(tab._group_of))
            step_of = {}
            for gi, stp in zip(tab._group_of, self._steps_np[tab._idx].tolist()):
                if step_of.setdefault(gi, stp) != stp:
                    raise MpoError(1, "graph step: parameters of one group at different step counts")
            hp_index = [groups.index(gi) for gi in tab._group_of]
            if hp_index != getattr(tab, "_hp_index", None):
                if ent is not None:
                    raise MpoError(1, "graph step: the group layout changed since capture")
                for i, h in enumerate(hp_index):
                    tab.arr[i].hp = h
                tab._hp_index = hp_index
            hps = [self._hp(self.param_groups[gi], max(1, step_of[gi])) for gi in groups]
            if ent is None:
                nb = api.hp_block_bytes(self._kind, self.exact)
                dev = params[0].device
                ent = self._graph[key] = {"tab": tab, "host": torch.empty(nb, dtype=torch.uint8, pin_memory=True),
                                          "dev": torch.empty(nb, dtype=torch.uint8, device=dev),
                                          "ack": torch.full((1,), -1, dtype=torch.int64, pin_memory=True)}
            ent["hps"] = hps
            api.hp_block_fill(self._kind, hps, ent["host"], seq=self._graph_seq, exact=self.exact)

    def _graph_step(self):
        if not self._graph:
            self._graph_tables(advance=False)      # first call (typically the capture): set up only
        ws = self._ws(self.param_groups[0]["params"][0].device) if self._needs_norm() else None
        for ent in self._graph.values():
            api.mpo_step_graphed(self._kind, ent["tab"], ent["hps"], ent["host"], ent["dev"], ack=ent["ack"],
                                 norm_ws=ws, exact=self.exact)

    # -- hook mode ---------------------------------------------------------------------------
    def install_backward_hooks(self, batch_below: int = 1 << 16, flush_elems: int = 1 << 22, native: bool = True):
        """Step each parameter inside backward, as soon as its gradient is accumulated, then free
        the gradient.  Returns the hook handles.

        Parameters smaller than ``batch_below`` elements (biases, norms) are not launched one by
        one: their gradients are held until ``flush_elems`` elements are pending or the backward
        ends, then stepped by one multi-tensor launch (bounded transient memory, far fewer
        launches).  ``batch_below=0`` steps every parameter individually; batching is off with
        ``skip_nonfinite`` (whose hook-mode skip is per parameter).  The hooks hold the optimizer
        weakly: keep a reference to it for as long as training runs.

        ``native=True`` (default): the hooks are C++ (csrc/mpo_hooks.cpp, autograd plumbing that
        calls the same C ABI): no Python runs per parameter, which keeps the hook mode's host cost
        per backward near the two-phase step's (P:104-111 report +3-4 % time).  ``native=False``:
        the same logic as Python hooks (A/B and reference)."""
        self._check_hook_mode()
        self._batch_below = 0 if self.skip_nonfinite else int(batch_below)
        self._flush_elems = int(flush_elems)
        if native:
            self._install_native()
            return []
        self._pending = []
        self._pending_elems = 0
        self._flush_queued = False
        self._hp_c, self._codes = {}, {}
        self._build_rows()
        if self.skip_nonfinite:
            n = sum(len(g["params"]) for g in self.param_groups)
            self._hook_S = torch.zeros(n, dtype=torch.float64, device=self.param_groups[0]["params"][0].device)
        for group in self.param_groups:
            for p in group["params"]:
                self._hooks.append(p.register_post_accumulate_grad_hook(_weak_hook(self)))
        return list(self._hooks)

    def _build_rows(self):
        self._rows = {}
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
                self._rows[p] = (row, gi)

    def _params_by_index(self):
        ps = [p for g in self.param_groups for p in g["params"]]
        return sorted(ps, key=lambda p: self.state[p]["index"])

    def _install_native(self):
        from . import _build, _lib
        if self._native is not None:
            raise MpoError(1, "native backward hooks are already installed")
        mod = _build.load_hooks()
        L = _lib.load(self.exact)
        fn = lambda name: C.cast(getattr(L, name), C.c_void_p).value
        params = self._params_by_index()
        dev = params[0].device
        ws = self._ws(dev) if self.skip_nonfinite else None
        bufs = (None, None)
        if self.skip_nonfinite:
            bufs = (torch.zeros(len(params), dtype=torch.float64, device=dev),
                    torch.zeros(len(params), dtype=torch.float64, pin_memory=True))
        ns = mod.HookState(self._kind, self.seed & 0xFFFFFFFFFFFFFFFF, self._batch_below, self._flush_elems,
                           self._steps.data_ptr(),
                           fn("mpo_fused_backward_hook_step"), fn("mpo_adam_step"), fn("mpo_sgd_step"),
                           fn("mpo_last_error"), 0 if ws is None else ws.data_ptr(),
                           0 if bufs[0] is None else bufs[0].data_ptr(), 0 if bufs[1] is None else bufs[1].data_ptr())
        gi_of = {id(p): gi for gi, g in enumerate(self.param_groups) for p in g["params"]}
        for p in params:
            st = self.state[p]
            ns.add_param(p.data.data_ptr(), st["resid"].data_ptr(), 0 if st.get("m") is None else st["m"].data_ptr(),
                         0 if st.get("v") is None else st["v"].data_ptr(), p.numel(), st["index"], gi_of[id(p)],
                         api.format_code(p.dtype, self.scheme))
        self._native, self._native_mod, self._native_bufs = ns, mod, bufs
        for gi in range(len(self.param_groups)):
            self.param_groups[gi] = _GroupDict(self.param_groups[gi], lambda gi=gi: self._push_group(gi))
            self._push_group(gi)
        for i, p in enumerate(params):
            mod.install(ns, p, i)
        self._native_fin = weakref.finalize(self, _native_finalize, ns, mod, [weakref.ref(p) for p in params])

    def _push_group(self, gi):
        if self._native is not None:
            self._native.set_group(gi, bytes(self._hp(self.param_groups[gi], 1).c()))

    def _pull_native_steps(self):
        """The native hooks count steps in place in self._steps; only a pending found-inf rollback
        of the last backward has to be applied before the counts are read."""
        if self._native is not None:
            self._native.resolve()


    def native_hook_calls(self) -> int:
        """Library calls the native hooks made so far (per-parameter steps + batched flushes)."""
        return 0 if self._native is None else int(self._native.calls())

    def remove_backward_hooks(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []
        if self._native is not None:
            self._pull_native_steps()
            self._native_fin()                       # disarm + uninstall
            self._native = None
            self.param_groups[:] = [dict(g) for g in self.param_groups]

    def _hook(self, p: torch.Tensor):
        if self._skip_check is not None:
            self._resolve_skips()          # the previous backward's skipped parameters
        st = self.state[p]
        g = p.grad
        self._steps_np[st["index"]] += 1
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
        row, group = self._rows[p]
        row.grad = g.data_ptr()
        # host cost per hook matters when backward is short: the ctypes hyper-parameters are built
        # once per (group, step) and shared by the group's parameters; format codes are cached
        key = (group, int(self._steps_np[st["index"]]))
        hp = self._hp_c.get(key)
        if hp is None:
            if len(self._hp_c) > 64:
                self._hp_c.clear()
            hp = self._hp_c[key] = self._hp(self.param_groups[group], key[1]).c()
        codes = self._codes.get((p.dtype, g.dtype))
        if codes is None:
            codes = self._codes[(p.dtype, g.dtype)] = (api.format_code(p.dtype, self.scheme), api.dtype_code(g.dtype))
        api.mpo_fused_backward_hook_step(self._kind, codes[0], codes[1], row, hp, exact=self.exact,
                                         norm_ws=self._ws(p.device) if self.skip_nonfinite else None)
        if self.skip_nonfinite:
            # this parameter's S (norm_ws[0] of its call) for the step-count rollback of a skip
            self._hook_S[st["index"]].copy_(self._norm_ws[0])
            if not self._flush_queued:
                torch.autograd.Variable._execution_engine.queue_callback(self._flush_pending)
                self._flush_queued = True
        p.grad = None   # freed now; stream order makes the block's reuse safe

    def _flush_pending(self, final: bool = True):
        """One multi-tensor launch over the batched small parameters of this backward."""
        if final:
            self._flush_queued = False
            if self._hook_S is not None:
                # end of backward: learn (later, without a sync) which parameters were skipped
                params = [p for g in self.param_groups for p in g["params"]]
                order = sorted(range(len(params)), key=lambda i: self.state[params[i]]["index"])
                self._queue_skip_check([params[i] for i in order], self._hook_S)
                self._hook_S.zero_()
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
                for p_, s_ in zip(ps, sts):
                    hp_index.append(keys.setdefault((self._rows[p_][1], int(self._steps_np[s_["index"]])), len(keys)))
                hps = [self._hp(self.param_groups[gi], stp) for (gi, stp) in keys]
                # one launch per MPO_MAX_HP_GROUPS (group, step) pairs (a launch's hyper-parameter bank)
                for c in range(0, len(hps), MPO_MAX_HP_GROUPS):
                    sel = [i for i, h in enumerate(hp_index) if c <= h < c + MPO_MAX_HP_GROUPS]
                    tab = api.TensorTable([ps[i].data for i in sel], [sts[i]["resid"] for i in sel],
                                          [items[i][1] for i in sel], [sts[i].get("m") for i in sel],
                                          [sts[i].get("v") for i in sel], [hp_index[i] - c for i in sel],
                                          scheme=self.scheme, sr_streams=[sts[i]["index"] for i in sel])
                    self._launch(tab, hps[c:c + MPO_MAX_HP_GROUPS])
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
        self._resolve_skips()
        if self._native is not None:
            self._native.resolve()
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
                 fmt: Optional[torch.dtype] = None, exact: bool = True, scheme: str = "rne", seed: int = 0,
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
                             weight_decay=g["weight_decay"], grad_scale=g["grad_scale"] * self._amp_inv, nesterov=g["nesterov"],
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
                 max_grad_norm: Optional[float] = None, fmt: Optional[torch.dtype] = None, exact: bool = True,
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
                              grad_scale=g["grad_scale"] * self._amp_inv, max_grad_norm=self.max_grad_norm, adamw=g["adamw"],
                              step=step, seed=api.step_seed(self.seed, step), clip_value=self.clip_value,
                              skip_nonfinite=self.skip_nonfinite)

    def _launch(self, tab, hps):
        ws = self._ws(tab.values[0].device) if (self.max_grad_norm > 0 or self.skip_nonfinite) else None
        api.mpo_adam_step(tab, hps, norm_ws=ws, exact=self.exact)

    def last_grad_sumsq(self) -> Optional[torch.Tensor]:
        """Device scalar: the fp64 sum of squares of the scaled gradients of the last clipped step."""
        return None if self._norm_ws is None else self._norm_ws[0]
