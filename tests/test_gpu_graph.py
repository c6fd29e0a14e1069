"""GPU: the CUDA-graph step (mpo_step_graphed, ResidualOptimizer.enable_graph_step).  The step's
per-step hyper-parameters -- bias corrections, lr from a schedule, SGD's first step, the
stochastic-rounding seed -- reach the captured kernels through a pinned host block copied at
execution time, so ONE capture replays every step; the result must equal the eager step() sequence
bitwise (exact build), with either step kernel, and when the whole training iteration (forward,
backward, optimizer) is one graph.
"""
import pytest
import torch
import torch.nn as nn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mpo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_12381_b200 as m
    from paper_2309_12381_b200 import _build
    _build.build()
    return m


def _opt(mpo, kind, ps, fmt, scheme="rne", clip=None):
    groups = [{"params": ps[::2]}, {"params": ps[1::2], "weight_decay": 0.0}]
    if kind == "adam":
        return mpo.ResidualAdamW(groups, lr=1e-3, betas=(0.9, 0.95), weight_decay=0.1, fmt=fmt, scheme=scheme, seed=4,
                                 max_grad_norm=clip)
    return mpo.ResidualSGD(groups, lr=0.05, momentum=0.9, weight_decay=1e-4, fmt=fmt, scheme=scheme, seed=4)


@pytest.mark.parametrize("kind,fmt,scheme,clip", [("adam", torch.bfloat16, "rne", None), ("adam", torch.float16, "sr", None),
                                                  ("adam", torch.bfloat16, "rne", 0.05), ("sgd", torch.float16, "rne", None),
                                                  ("sgd", torch.bfloat16, "x8z", None), ("adam", torch.float16, "x8", None)])
def test_graph_step_equals_eager(mpo, step_kernel, kind, fmt, scheme, clip):
    """Only opt.step() captured; gradients copied into their (static) buffers before each replay;
    an LR schedule changes group 0's lr every step.  6 replays == 6 eager steps, bitwise."""
    torch.manual_seed(1)
    shapes = [(300, 17), (4096,), (5,), (64, 128), (1000,)]
    src = [torch.randn(s, device="cuda") * 0.02 for s in shapes]
    grads = [[(torch.randn(s, device="cuda") * 1e-2).to(fmt) for s in shapes] for _ in range(6)]
    pa = [nn.Parameter(t.clone()) for t in src]
    pb = [nn.Parameter(t.clone()) for t in src]
    oa, ob = _opt(mpo, kind, pa, fmt, scheme, clip), _opt(mpo, kind, pb, fmt, scheme, clip)
    for p in pb:
        p.grad = torch.zeros(p.shape, dtype=fmt, device="cuda")
    ob.enable_graph_step()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ob.step()                                     # captured, nothing executed
    for t in range(6):
        lr = 1e-3 * (0.7 ** t) if kind == "adam" else 0.05 * (0.7 ** t)
        oa.param_groups[0]["lr"] = ob.param_groups[0]["lr"] = lr
        for p, gg in zip(pa, grads[t]):
            p.grad = gg.clone()
        oa.step()
        for p, gg in zip(pb, grads[t]):
            p.grad.copy_(gg)
        ob.prepare_step()
        g.replay()
    torch.cuda.synchronize()
    for x, y in zip(pa, pb):
        assert torch.equal(x.view(torch.int16), y.view(torch.int16))
        sx, sy = oa.state[x], ob.state[y]
        assert torch.equal(sx["resid"], sy["resid"]) and int(sx["step"]) == int(sy["step"]) == 6
        for k in ("m", "v"):
            if sx.get(k) is not None:
                assert torch.equal(sx[k], sy[k])


def test_whole_iteration_graph_equals_eager(mpo):
    """Forward + backward + the residual AdamW step captured as ONE CUDA graph and replayed (static
    input buffer) == the same iterations run eagerly, bitwise."""
    torch.manual_seed(2)
    d = 128

    def mk():
        return nn.Sequential(nn.Linear(d, 4 * d), nn.GELU(), nn.Linear(4 * d, d)).cuda()
    a, b = mk(), mk()
    b.load_state_dict(a.state_dict())
    oa = mpo.ResidualAdamW(a.parameters(), lr=1e-3, weight_decay=0.1, fmt=torch.bfloat16)
    ob = mpo.ResidualAdamW(b.parameters(), lr=1e-3, weight_decay=0.1, fmt=torch.bfloat16)
    xs = [torch.randn(32, d, device="cuda", dtype=torch.bfloat16) for _ in range(5)]

    def loss_of(m, x):
        return m(x).float().square().mean()
    # warm-up on a side stream so every parameter owns its gradient buffer (then keep them: no
    # set_to_none), as torch's graph-capture recipe prescribes
    x_static = torch.zeros(32, d, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        loss_of(b, x_static).backward()
    torch.cuda.current_stream().wait_stream(s)
    for p in b.parameters():
        p.grad.zero_()
    ob.enable_graph_step()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for p in b.parameters():
            p.grad.zero_()
        loss_of(b, x_static).backward()
        ob.step()
    for x in xs:
        loss_of(a, x).backward()
        oa.step()
        for p in a.parameters():
            p.grad = None
        x_static.copy_(x)
        ob.prepare_step()
        g.replay()
    torch.cuda.synchronize()
    for pa_, pb_ in zip(a.parameters(), b.parameters()):
        assert torch.equal(pa_.view(torch.int16), pb_.view(torch.int16))
