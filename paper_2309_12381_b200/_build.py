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
FORMATS = (0, 1, 16, 17, 32, 48, 49)
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


def build(force: bool = False, verbose: bool = False):
    """Compile both libraries if a source is newer than the output."""
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
    return outs


if __name__ == "__main__":
    for p in build(force="--force" in sys.argv, verbose=False):
        print(p)
