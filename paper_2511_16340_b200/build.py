"""Builds libwarmgp_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The library is the product: hand-written CUDA kernels + the C-ABI of
include/warmgp_capi.h.  Objects go to build/, the shared library next to this file
so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "warmgp_b200")
LIB = os.path.join(HERE, "libwarmgp_b200.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
          "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "warmgp_capi.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, verbose: bool, build_dir: str = BUILD, extra=()) -> str:
    obj = os.path.join(build_dir, src + ".o")
    path = os.path.join(CSRC, src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), _headers_mtime()):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", path, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def _nccl_link() -> list:
    """Link NCCL from the torch-bundled wheel when present (the same libnccl.so.2 soname
    torch loads: whichever of torch and this library loads first, the process then holds
    one NCCL that both can use -- the system 2.27 lacks symbols torch 2.11 needs), else the
    system library."""
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
        dirs = [os.path.join(p, "lib") for p in (spec.submodule_search_locations or [])] if spec else []
    except Exception:  # noqa: BLE001
        dirs = []
    for d in dirs:
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return ["-L" + d, "-l:libnccl.so.2", "-Xlinker", "-rpath," + d,
                    "-Xlinker", "-rpath,/usr/lib/x86_64-linux-gnu"]
    return ["-lnccl", "-Xlinker", "-rpath,/usr/lib/x86_64-linux-gnu"]


def build(verbose: bool = False, extra=(), lib: str = LIB, build_dir: str = BUILD) -> str:
    """Compile every source and link ``lib``.  ``extra`` nvcc flags (e.g. -D switches of A/B
    probe variants) go with a separate ``build_dir`` and ``lib``."""
    os.makedirs(build_dir, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, build_dir, tuple(extra)), srcs))
    if os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(o) for o in objs):
        return lib
    cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, *_nccl_link()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    # python -m paper_2511_16340_b200.build [-v] [--variant NAME -DFLAG ...]: a variant
    # library tools/probes/_variants/libwarmgp_NAME.so for A/B probes (WGP_LIB_PATH)
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        name, flags = args[i + 1], [a for a in args[i + 2:] if a.startswith("-D")]
        vdir = os.path.join(ROOT, "tools", "probes", "_variants")
        os.makedirs(vdir, exist_ok=True)
        print(build(verbose="-v" in args, extra=flags, lib=os.path.join(vdir, f"libwarmgp_{name}.so"),
                    build_dir=os.path.join(ROOT, "build", f"variant_{name}")))
    else:
        print(build(verbose="-v" in args))
