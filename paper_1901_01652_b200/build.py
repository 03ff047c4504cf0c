"""Build libtrg.so in-tree for sm_100a (B200).

    python -m paper_1901_01652_b200.build        (or __graft_entry__.build())

Each CUDA / C++ source is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
paper_1901_01652_b200/libtrg.so (git-ignored, travels to the GPU box with
gpurun). Objects are rebuilt only when a source or header is newer.
"""
import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libtrg.so")

SOURCES = ["sketch.cu", "stream_f64.cu", "slab_f64.cu", "slab_tma.cu", "stream_f32.cu", "tc_f32.cu", "slab_f32.cu", "slab_st.cu", "ttm.cu", "qr.cu", "tr.cu", "runtime.cpp", "host_solve.cpp", "device_ls.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _flags():
    return ARCH + [
        "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
        "-Xcompiler", "-fPIC,-fopenmp,-O3,-march=x86-64-v4",
        "-Xptxas", "-v" if os.environ.get("TRG_PTXAS_VERBOSE") else "-O3",
        "-ccbin", "g++",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
    ] + os.environ.get("TRG_EXTRA_NVCC", "").split()


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".hpp", ".cuh"))]
    return hs + [os.path.join(ROOT, "include", "trg.h")]


def _newer(src, dst, deps):
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(p) > t for p in [src] + deps)


def build(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    deps = _headers()
    objs, cmds = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if _newer(src, obj, deps):
            cmds.append([NVCC] + _flags() + ["-c", src, "-o", obj])
    # one nvcc per translation unit, in parallel (each is single-threaded)
    jobs = max(1, min(len(cmds), os.cpu_count() or 1))
    with concurrent.futures.ThreadPoolExecutor(jobs) as ex:
        for cmd, rc in zip(cmds, ex.map(lambda c: (print(" ".join(c), flush=True) if verbose else None,
                                                   subprocess.run(c).returncode)[1], cmds)):
            if rc != 0:
                raise subprocess.CalledProcessError(rc, cmd)
    if any(_newer(o, LIB, []) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-Xcompiler", "-fopenmp", "-ldl", "-lgomp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    print(LIB)
