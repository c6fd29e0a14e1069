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
SOURCES = [os.path.join(CSRC, "mpo.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "mpo_device.cuh"), os.path.join(INCLUDE, "mpo.h"), __file__]

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


def flags(exact: bool):
    inc, lib = nccl_dirs()
    f = ["-std=c++17", "-O3", *ARCH, "-lineinfo", "-shared", "-Xcompiler",
         "-fPIC,-fvisibility=hidden,-ffp-contract=off", "-ftz=false", "-prec-div=true",
         "-prec-sqrt=true", "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{inc}", f"-L{lib}",
         "-l:libnccl.so.2", f"-Xlinker", f"-rpath,{lib}"]
    f += ["-fmad=false", "-DMPO_EXACT"] if exact else ["-fmad=true"]
    return f


def build_variant(name: str, defines, exact: bool = False) -> str:
    """Build an experimental variant (extra -D defines) into lib/variants/ (A/B measurements)."""
    out = os.path.join(LIBDIR, "variants", f"libmpo_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *flags(exact), *[f"-D{d}" for d in defines], "-o", out, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building variant {name}")
    return out


def lib_path(exact: bool = False) -> str:
    return os.path.join(LIBDIR, "libmpo_exact.so" if exact else "libmpo.so")


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
            tmp = out + f".tmp{os.getpid()}"
            cmd = [NVCC, *flags(exact), "-o", tmp, *SOURCES]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
            with open(out + ".ptxas.txt", "w") as fh:
                fh.write(r.stderr)
            if verbose:
                sys.stderr.write(r.stderr)
            os.replace(tmp, out)
        outs.append(out)
    return outs


if __name__ == "__main__":
    for p in build(force="--force" in sys.argv, verbose=True):
        print(p)
