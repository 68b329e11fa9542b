"""Builds libmrq.so in-tree for sm_100a (nvcc; no JIT cache).

Each csrc/*.cu compiles to its own object under build/ (in parallel; an
object is rebuilt when its source or any header is newer), then nvcc links
the shared library.  MRQ_NVCC_EXTRA adds flags (A/B variant builds); objects
built with other extra flags are rebuilt (the flags are part of their name).
"""
import glob
import hashlib
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libmrq.so")
SRC = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HDR = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(HERE, "..", "include", "mrq.h")]
OBJ_DIR = os.path.join(HERE, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


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


def _flags():
    inc, lib = nccl_paths()
    f = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC"]
    if inc:
        # headers only: NCCL itself is dlopen'ed at run time (csrc/mrq_comm.cu)
        f += ["-DMRQ_HAVE_NCCL=1", "-I", inc, '-DMRQ_NCCL_LIB="%s"' % os.path.join(lib, "libnccl.so.2")]
    return f + os.environ.get("MRQ_NVCC_EXTRA", "").split()


def _obj(src, flags):
    tag = hashlib.sha1(" ".join(flags).encode()).hexdigest()[:8]
    return os.path.join(OBJ_DIR, os.path.basename(src)[:-3] + "." + tag + ".o")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SRC + HDR)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJ_DIR, exist_ok=True)
    flags = _flags() + (["-Xptxas", "-v"] if verbose else [])
    hdr_t = max(os.path.getmtime(h) for h in HDR)

    def comp(src):
        o = _obj(src, flags)
        if (force and force != "relink") or not os.path.exists(o) or \
                os.path.getmtime(o) < max(os.path.getmtime(src), hdr_t):
            subprocess.check_call(["nvcc"] + flags + ["-c", src, "-o", o + ".tmp"])
            os.replace(o + ".tmp", o)
        return o

    with ThreadPoolExecutor(max_workers=min(8, len(SRC))) as ex:
        objs = list(ex.map(comp, SRC))
    subprocess.check_call(["nvcc"] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-ldl"])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
