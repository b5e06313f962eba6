"""Build libdem.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libdem.so")
SOURCES = ["ctx.cu", "detect.cu", "solve.cu", "sweep.cu", "dist.cu", "generate.cu", "gs.cu", "scan.cu", "radix_sort.cu", "planner.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr"]


DEFAULT_DEFINES = ("DEM_G64", "DEM_R64")


def build(force=False, verbose=False, defines=DEFAULT_DEFINES, out=None):
    OUT_ = out or OUT
    os.makedirs(os.path.dirname(OUT_), exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "dem.h")]
    if not force and os.path.exists(OUT_) and os.path.getmtime(OUT_) >= max(os.path.getmtime(d) for d in deps):
        return OUT_
    tag = "_".join(d.lower() for d in defines)
    objdir = os.path.join(HERE, "lib", "obj_" + (tag or "fp32"))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in SOURCES:
        o = os.path.join(objdir, s + ".o")
        cmd = [NVCC] + FLAGS + ["-D" + d for d in defines] + ["-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.check_call(cmd)
        objs.append(o)
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", OUT_] + objs +
                          ["-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    return OUT_


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
