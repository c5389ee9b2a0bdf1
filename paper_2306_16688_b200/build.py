"""Build libsrl.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo).

    python -m paper_2306_16688_b200.build [--force] [-v]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
SO = os.path.join(HERE, "libsrl.so")
SOURCES = ["gae.cu", "mlp.cu", "misc.cu", "api.cu", "head_fused.cu"]
HEADERS = ["ptx.cuh", "gemm_tc.cuh", "internal.h"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("torch's NCCL wheel (nvidia.nccl) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> str:
    """defines: extra -D flags (tools/build_variant.py); out: alternative .so path."""
    inc, lib = nccl_dirs()
    build_dir = BUILD if out is None else os.path.join(os.path.dirname(out), "obj")
    so = SO if out is None else out
    os.makedirs(build_dir, exist_ok=True)
    hdr = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "srl.h")]
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                    "-I", CSRC, "-I", inc, "--expt-relaxed-constexpr"] + [f"-D{d}" for d in defines]
    if verbose:
        flags += ["-Xptxas", "-v"]

    def compile_one(src):
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        if force or _stale(o, [s] + hdr):
            cmd = [nvcc()] + flags + ["-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
            if verbose:
                sys.stderr.write(r.stderr)
        return o

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or _stale(so, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "shared", "-o", so] + objs + [
            "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}",
            "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
