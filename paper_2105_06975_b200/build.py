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
    # one nvcc per translation unit, run concurrently (no cross-file device code, so
    # whole-program compilation is not needed), then one host link
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    # WF4DVAR_NVCC_FLAGS: extra flags for tuning experiments (e.g. -DL96_MINB_F=2); pass
    # force=True when they change (object files are reused by modification time only)
    ccmd = [_nvcc(), ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
            "-Xptxas", "-v" if verbose else "-O3"] + os.environ.get("WF4DVAR_NVCC_FLAGS", "").split() + ["-c"]
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]

    def _one(so):
        src, obj = so
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
                [os.path.getmtime(src)] + [os.path.getmtime(h) for h in hdrs if os.path.exists(h)]):
            return None
        r = subprocess.run(ccmd + ["-o", obj + ".tmp", src], capture_output=True, text=True)
        if r.returncode == 0:
            os.replace(obj + ".tmp", obj)
        return r

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(srcs), max(1, os.cpu_count() or 1))) as ex:
        results = list(ex.map(_one, zip(srcs, objs)))
    for src, r in zip(srcs, results):
        if r is None:
            continue
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed compiling " + os.path.basename(src))
        if verbose:
            sys.stderr.write(r.stderr)
    cmd = [_nvcc(), ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB + ".tmp"] + objs + [
           "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcusolver", "-lcublas", "-ldl",
           "-Xlinker", "-rpath=" + os.path.join(CUDA_HOME, "lib64")]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libwf4dvar.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(LIB)
