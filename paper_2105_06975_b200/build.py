"""In-tree build of the C-ABI shared library libwf4dvar.so for sm_100a.

    python -m paper_2105_06975_b200.build        # or __graft_entry__.build()

nvcc cross-compiles here without a GPU; the .so lands next to this file so it
travels to the GPU box with the repo snapshot.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libwf4dvar.so")
SOURCES = ["api.cu", "saddle.cu", "gemm.cu", "trsm.cu", "model.cu", "l96.cu", "vec.cu", "krylov.cu", "comm.cu", "spectral.cu", "outer.cu", "sparse.cu"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _nvcc():
    p = os.path.join(CUDA_HOME, "bin", "nvcc")
    return p if os.path.exists(p) else "nvcc"


def build(verbose=False, force=False):
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(HERE, "..", "include", "wf4dvar.h"))
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(f) <= t for f in srcs + hdrs if os.path.exists(f)):
            return LIB
    cmd = [_nvcc(), ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-Xptxas", "-v" if verbose else "-O3",
           "-o", LIB + ".tmp"] + srcs + [
           "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcusolver", "-lcublas", "-ldl",
           "-Xlinker", "-rpath=" + os.path.join(CUDA_HOME, "lib64")]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libwf4dvar.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(LIB)
