"""In-tree build of libfic_b200.so (sm_100a) with nvcc.

    python -m paper_1404_0774_b200.build [--force]

The shared library is written next to this file so it travels with the repo snapshot
to the GPU box; nothing is JIT-compiled at import time.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("FIC_LIB") or os.path.join(HERE, "libfic_b200.so")
SOURCES = ["fic_api.cu", "pool.cu", "matcher_simt.cu", "scan.cu", "decoder.cu", "fit.cu", "fic1.cu"]
HEADERS = ["common.cuh", "tc_ptx.cuh", os.path.join("..", "..", "include", "fic_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
         "-Xptxas", "-warn-spills"] + (["-DFIC_TRACE"] if os.environ.get("FIC_TRACE") else [])  # pipeline trace build
FLAGS += os.environ.get("FIC_NVCC_DEFINES", "").split()  # experiments, e.g. "-DFIC_EVAL_MINB_FULL=3"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "_obj" + ("_" + os.path.basename(LIB) if os.environ.get("FIC_LIB") else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        o = os.path.join(objdir, s.replace(".cu", ".o"))
        cmd = [NVCC] + ARCH + FLAGS + ["-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            print(" ".join(cmd))
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), s))
        objs.append(o)
    failed = []
    for p, s in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            failed.append(s)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
