"""Builds libmrq.so in-tree for sm_100a (nvcc; no JIT cache)."""
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libmrq.so")
SRC = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HDR = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(HERE, "..", "include", "mrq.h")]


def nccl_paths():
    try:
        import nvidia.nccl as nn
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    except Exception:  # pragma: no cover
        return None, None
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")):
        return inc, lib
    return None, None


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SRC + HDR)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    inc, lib = nccl_paths()
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
           "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", LIB + ".tmp"] + SRC
    if inc:
        # headers only: NCCL itself is dlopen'ed at run time (csrc/mrq_comm.cu)
        cmd += ["-DMRQ_HAVE_NCCL=1", "-I", inc, '-DMRQ_NCCL_LIB="%s"' % os.path.join(lib, "libnccl.so.2")]
    cmd += ["-ldl"] + os.environ.get("MRQ_NVCC_EXTRA", "").split()   # A/B variant builds (scripts/variant.sh)
    if verbose:
        cmd += ["-Xptxas", "-v"]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
