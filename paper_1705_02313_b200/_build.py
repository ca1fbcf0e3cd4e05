"""Build libpgsi.so (nvcc, sm_100a) in-tree. Used by __graft_entry__.build()."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpgsi.so")
SOURCES = ["pg_api.cu", "pg_kernels.cu", "pg_bf.cu", "pg_small.cu", "pg_verify.cu", "pg_trace.cu", "pg_loop.cu", "pg_load_dev.cu", "pg_load.cpp", "pg_io.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def nccl_dirs():
    """(include, lib) of the NCCL that torch loads (nvidia-nccl wheel), else the system's."""
    try:
        import nvidia.nccl as nn
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except ImportError:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    """extra: additional nvcc flags (e.g. -D defines for A/B variants written to `out`)."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "pg_internal.cuh"), os.path.join(ROOT, "include", "pg.h")]
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB
    ninc, nlib = nccl_dirs()
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"), "-I", ninc,
           *extra, "-o", out + ".tmp", *srcs, "-L", nlib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nlib}"]
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python _build.py [-v] [-o OUT.so] [-DNAME=VAL ...]
    import sys
    a = sys.argv[1:]
    out = a[a.index("-o") + 1] if "-o" in a else LIB
    print(build(force=True, verbose="-v" in a, out=os.path.abspath(out), extra=[x for x in a if x.startswith("-D")]))
