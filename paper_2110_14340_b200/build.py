"""In-tree build of libjacc.so (sm_100a SASS; no PTX JIT needed on the box).

nvcc compiles the device kernels, g++ the host runtime; the shared library
links CUDA's static runtime and the NCCL that ships with the torch wheel
(one libnccl.so.2 per process, found through an rpath)."""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libjacc.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# host runtime translation units (all share csrc/rt.hpp)
HOST = ("abi.cpp", "plan.cpp", "launch.cpp", "mp.cpp", "graphs.cpp")
SOURCES = [os.path.join(CSRC, f) for f in ("kernels.cu", "kernels.cuh", "rt.hpp") + HOST] + [
    os.path.join(INCLUDE, "jacc.h"), os.path.join(CSRC, "exports.map")]


def nccl_paths():
    import nvidia.nccl as nn  # the wheel torch itself loads
    base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"libjacc build failed at {os.path.basename(cmd[0])}")
    return r


def build(force=False, verbose=False, defines=(), out=None):
    """defines / out: experiment builds (tools/) -- extra -D flags for the
    kernels, written to `out` instead of the package's libjacc.so."""
    if defines or out:
        force = True
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(s) <= t for s in SOURCES):
            return LIB
    nccl_inc, nccl_lib = nccl_paths()
    bdir = os.path.join(PKG, "_build") if not (defines or out) else (out + ".build")
    os.makedirs(bdir, exist_ok=True)
    ko = os.path.join(bdir, "kernels.o")
    _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines], "-I", INCLUDE, "-c",
          os.path.join(CSRC, "kernels.cu"), "-o", ko])
    objs = [ko]
    for src in HOST:
        o = os.path.join(bdir, src.replace(".cpp", ".o"))
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", *[f"-D{d}" for d in defines], "-I", INCLUDE,
              "-I", os.path.join(CUDA_HOME, "include"), "-I", nccl_inc, "-c",
              os.path.join(CSRC, src), "-o", o])
        objs.append(o)
    dst = out or LIB
    tmp = dst + ".tmp"
    # only the jacc_* C-ABI is exported (csrc/exports.map)
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static",
          "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}",
          "-Xlinker", f"--version-script={os.path.join(CSRC, 'exports.map')}"])
    os.replace(tmp, dst)
    return dst


if __name__ == "__main__":
    # python build.py [-v] [--out PATH] [-DNAME=VAL ...]
    a = sys.argv[1:]
    o = a[a.index("--out") + 1] if "--out" in a else None
    print(build(force=True, verbose="-v" in a, defines=[x[2:] for x in a if x.startswith("-D")], out=o))
