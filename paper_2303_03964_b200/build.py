"""Builds libtfdp.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the
repo snapshot to the GPU box).  Usage: python -m paper_2303_03964_b200.build [-v]"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtfdp.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        inc = os.path.join(base, "nccl", "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    for inc in ("/usr/include", "/usr/local/cuda/include"):
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel or system NCCL headers)")


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps.append(os.path.join(ROOT, "include", "tfdp.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), out: str = None) -> str:
    """Compiles every source to an object in parallel (one nvcc per file), then links.
    defines / out: developer A/B variants (e.g. -DTFDP_ATTR_BATCH=4 into another .so)."""
    out = out or LIB
    if not force and out == LIB and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    common = [
        _nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo",
        "-Xcompiler", "-fPIC,-fopenmp,-O3",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", _nccl_include(),
        *(["-Xptxas", "-v"] if verbose else []),
        *defines,
    ]
    objdir = os.path.join(ROOT, "build", "obj" if out == LIB else "obj_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = common + ["-c", src, "-o", obj]
        return obj, cmd, subprocess.run(cmd, capture_output=True, text=True)

    srcs = sources()
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, srcs))
    for obj, cmd, r in results:
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd))
    cmd = [_nvcc(), *ARCH, "--shared", "-Xcompiler", "-fPIC,-fopenmp",
           *[o for o, _, _ in results], "-lgomp", "-ldl", "-o", out + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + " ".join(cmd))
    os.replace(out + ".tmp", out)
    if out == LIB:
        build_examples(verbose)
        try:  # test infrastructure: never fails the product build
            build_nccl_loopback(verbose)
        except Exception as e:  # noqa: BLE001
            sys.stderr.write(f"[build] tests/nccl_loopback not built: {e}\n")
    return out


EXAMPLES = os.path.join(ROOT, "examples")


def build_examples(verbose: bool = False) -> list:
    """Plain C clients of the C ABI (examples/*.c), linked against the in-tree libtfdp.so."""
    outs = []
    for src in sorted(glob.glob(os.path.join(EXAMPLES, "*.c"))):
        exe = os.path.splitext(src)[0]
        cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-L", HERE,
               "-ltfdp", "-Wl,-rpath,$ORIGIN/../paper_2303_03964_b200", "-lm", "-o", exe]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError("gcc failed:\n" + " ".join(cmd))
        outs.append(exe)
    return outs


LOOPBACK_SRC = os.path.join(ROOT, "tests", "nccl_loopback", "nccl_loopback.cpp")
LOOPBACK_LIB = os.path.join(ROOT, "tests", "nccl_loopback", "libnccl_loopback.so")


def build_nccl_loopback(verbose: bool = False) -> str:
    """The tests' in-process NCCL stand-in (TFDP_NCCL_LIB; test infrastructure, not linked
    into libtfdp.so): g++ against the CUDA runtime."""
    cuda = os.path.dirname(os.path.dirname(_nvcc()))
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(cuda, "include"),
           "-I", _nccl_include(), LOOPBACK_SRC, "-L", os.path.join(cuda, "lib64"), "-lcudart",
           "-Wl,-rpath," + os.path.join(cuda, "lib64"), "-o", LOOPBACK_LIB]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("g++ failed:\n" + " ".join(cmd))
    return LOOPBACK_LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
