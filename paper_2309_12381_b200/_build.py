"""In-tree build of the CUDA library (sm_100a only).

Two shared libraries are produced from the same sources:

* ``lib/libmpo.so``       default FMA contraction (the product build);
* ``lib/libmpo_exact.so`` ``-fmad=false``: bit-exact to the CPU oracle.

Both always use IEEE division/sqrt and keep subnormals (``-ftz=false -prec-div=true
-prec-sqrt=true``; ``--use_fast_math`` is never used).  NCCL is linked from the torch wheel so
that the communicator borrowed from ``ProcessGroupNCCL`` belongs to the same libnccl.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
INCLUDE = os.path.join(ROOT, "include")
# translation units: the ABI layer, and the step kernels once per storage format (mpo_dtype code)
ABI_TU = os.path.join(CSRC, "mpo.cu")
INST_TU = os.path.join(CSRC, "mpo_inst.cu")
FORMATS = (0, 1, 16, 17, 32, 48, 49, 64, 65)
SOURCES = [ABI_TU, INST_TU]
DEPS = SOURCES + [os.path.join(CSRC, "mpo_device.cuh"), os.path.join(CSRC, "mpo_kernels.cuh"),
                  os.path.join(INCLUDE, "mpo.h"), __file__]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("NCCL headers/library from the torch wheel (nvidia/nccl) not found")


def compile_flags(exact: bool):
    inc, _ = nccl_dirs()
    f = ["-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
         "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{inc}"]
    f += ["-fmad=false", "-DMPO_EXACT"] if exact else ["-fmad=true"]
    return f


def link_flags():
    _, lib = nccl_dirs()
    return ["-shared", *ARCH, f"-L{lib}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]


def lib_path(exact: bool = False) -> str:
    return os.path.join(LIBDIR, "libmpo_exact.so" if exact else "libmpo.so")


def _compile_link(out: str, exact: bool, defines=()):
    """Compile every translation unit in parallel, then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    objdir = out + ".obj"
    os.makedirs(objdir, exist_ok=True)
    jobs = [(ABI_TU, os.path.join(objdir, "mpo.o"), [])]
    jobs += [(INST_TU, os.path.join(objdir, f"inst_{sf}.o"), [f"-DMPO_SF={sf}"]) for sf in FORMATS]

    def one(job):
        src, obj, extra = job
        cmd = [NVCC, *compile_flags(exact), *[f"-D{d}" for d in defines], *extra, "-c", "-o", obj, src]
        return subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(one, jobs))
    log = "".join(r.stdout + r.stderr for r in results)
    if any(r.returncode != 0 for r in results):
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
    tmp = out + f".tmp{os.getpid()}"
    r = subprocess.run([NVCC, *link_flags(), "-o", tmp, *[j[1] for j in jobs]], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"link failed for {os.path.basename(out)}")
    os.replace(tmp, out)
    return log


def build_variant(name: str, defines, exact: bool = False) -> str:
    """Build an experimental variant (extra -D defines) into lib/variants/ (A/B measurements)."""
    out = os.path.join(LIBDIR, "variants", f"libmpo_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    _compile_link(out, exact, defines)
    return out


def _stale(out: str) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in DEPS)


HOOKS_SRC = os.path.join(CSRC, "mpo_hooks.cpp")


def hooks_path() -> str:
    import sysconfig
    return os.path.join(LIBDIR, "mpo_hooks" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_hooks(force: bool = False) -> str:
    """The native post-accumulate-grad hook module (csrc/mpo_hooks.cpp: autograd plumbing that
    calls the C ABI; no kernels), compiled with g++ against the installed torch -- in-tree, so it
    travels with the repository like the CUDA libraries."""
    import sysconfig
    import torch
    from torch.utils import cpp_extension as ce
    out = hooks_path()
    deps = [HOOKS_SRC, os.path.join(INCLUDE, "mpo.h"), __file__]
    if not force and os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out) for d in deps):
        return out
    inc = ce.include_paths(device_type="cuda") + [sysconfig.get_paths()["include"], INCLUDE]
    libs = ce.library_paths(device_type="cuda")
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden", "-w",
           f"-D_GLIBCXX_USE_CXX11_ABI={abi}", "-DTORCH_EXTENSION_NAME=mpo_hooks", "-DTORCH_API_INCLUDE_EXTENSION_H",
           *[f"-I{d}" for d in inc], HOOKS_SRC, *[f"-L{d}" for d in libs],
           "-lc10", "-lc10_cuda", "-ltorch", "-ltorch_cpu", "-ltorch_python", "-lcudart",
           *[f"-Wl,-rpath,{d}" for d in libs], "-o", out + f".tmp{os.getpid()}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building the native hook module")
    os.replace(out + f".tmp{os.getpid()}", out)
    return out


def load_hooks():
    """Import the native hook module from lib/ (ImportError if it was not built)."""
    import importlib.util
    path = hooks_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_2309_12381_b200._build`")
    import torch  # noqa: F401  (the module links against torch's libraries)
    spec = importlib.util.spec_from_file_location("mpo_hooks", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def build(force: bool = False, verbose: bool = False):
    """Compile both libraries (and the native hook module) if a source is newer than the output."""
    os.makedirs(LIBDIR, exist_ok=True)
    outs = []
    for exact in (False, True):
        out = lib_path(exact)
        if force or _stale(out):
            log = _compile_link(out, exact)
            with open(out + ".ptxas.txt", "w") as fh:
                fh.write(log)
            if verbose:
                sys.stderr.write(log)
        outs.append(out)
    outs.append(build_hooks(force))
    return outs


if __name__ == "__main__":
    for p in build(force="--force" in sys.argv, verbose=False):
        print(p)
