"""bench.py's own arm on the GPU: one JSON line with every key the driver reads, the roofline and
clock blocks filled, the e2e leg's copies declared, and this library's launches counted."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "resnet50_sgd", "--steps", "5",
                        "--warmup", "3", "--no-secondary", "--no-cpu-baseline", "--e2e-steps", "3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[:2000]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["gpu_launches"] == 5                        # one step-kernel launch per timed step
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
    assert abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    assert rf["algorithmic_bytes_per_launch"] == 18 * 25557032
    assert d["clocks"]["sm_max_mhz"] and d["clocks"]["samples"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == json.loads(json.dumps(bench.workload_config("resnet50_sgd")))


def test_bench_multi_gpu_breakdown_path_at_world1():
    """The N > 1 code path of the bench at world 1 (--mg-breakdown; the fused P2P step through the
    child-process route with MPO_BENCH_FUSED_CHILD=1): update-only timing, the two collectives'
    busbw fields and the fused step all present, none of them an error."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ, MPO_BENCH_FUSED_CHILD="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "gpt2_adamw", "--steps", "4",
                        "--warmup", "3", "--no-secondary", "--no-cpu-baseline", "--e2e-steps", "2", "--mg-breakdown"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    mg = d["multi_gpu"]
    assert "error" not in json.dumps(mg), json.dumps(mg)[:2000]
    assert mg["update_only"]["ms_per_step"] > 0
    for k in ("reduce_scatter_grad16", "all_gather_value16"):
        assert k in mg and mg[k]["ms"] > 0
    assert mg["p2p_fused_step"]["ms_per_step"] > 0 and mg["p2p_fused_step"]["launches_per_step"] == 1
