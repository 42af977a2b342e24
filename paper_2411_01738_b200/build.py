"""Build libxdit_usp.so in-tree: nvcc for the sm_100a kernels, g++ for the host orchestrator,
linked against the NCCL that torch ships (2.28.x, ABI-compatible with torch's communicators).

    python -m paper_2411_01738_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libxdit_usp.so")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    """(include, lib) of the NCCL bundled with torch (nvidia-nccl-cu12 wheel)."""
    cands = []
    try:
        import nvidia.nccl as m  # type: ignore
        cands += [os.path.dirname(m.__file__)] if getattr(m, "__file__", None) else list(m.__path__)
    except Exception:
        pass
    cands.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl"))
    for c in cands:
        inc, lib = os.path.join(c, "include"), os.path.join(c, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("torch's NCCL (nvidia/nccl/{include,lib}) not found")


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False, defines=(), tag: str | None = None) -> str:
    """Build the library.  `defines`/`tag`: kernel A/B experiments -- extra -D flags, objects in
    _build_<tag>/ and the library as libxdit_usp_<tag>.so (load it with XDIT_LIB=<path>)."""
    BUILD = os.path.join(HERE, "_build" + (f"_{tag}" if tag else ""))
    LIB = os.path.join(HERE, f"libxdit_usp_{tag}.so" if tag else "libxdit_usp.so")
    os.makedirs(BUILD, exist_ok=True)
    inc, lib = nccl_dirs()
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(INCLUDE, "xdit_usp.h")]
    objs = []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [src] + headers):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler",
                   "-fvisibility=hidden", *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", inc, "-c", src,
                   "-o", obj]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-Wall",
                   "-I", INCLUDE, "-I", inc, "-I", os.path.join(CUDA_HOME, "include"), "-c", src, "-o", obj]
        _run(cmd)
    if force or _stale(LIB, objs):
        # exported symbols = the extern "C" entry points (default visibility via a version script)
        vs = os.path.join(BUILD, "exports.map")
        with open(vs, "w") as f:
            f.write("{ global: xdit_*; local: *; };\n")
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
              "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}",
              "-Xlinker", f"--version-script={vs}"])
    return LIB


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    tag = next((a.split("=", 1)[1] for a in args if a.startswith("--tag=")), None)
    build(force="--force" in args, verbose_ptxas="-v" in args, defines=defs, tag=tag)
