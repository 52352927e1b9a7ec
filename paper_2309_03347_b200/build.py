"""Build libtt.so in-tree for sm_100a (nvcc, -lineinfo).  Used by
__graft_entry__.build() and the tests; the .so travels to the GPU box with
the repo snapshot."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libtt.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-O3"] + os.environ.get("TT_NVCC_EXTRA", "").split()   # experiments only


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(INC, "tt.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, jobs=8):
    if not force and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = ["nvcc", *ARCH, *FLAGS, "-I", INC, "-I", CSRC, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        if len(procs) >= jobs:
            _drain(procs)
    _drain(procs)
    cmd = ["nvcc", *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("link failed:\n" + out.stdout + out.stderr)
    build_launch_counter()
    return LIB


LC_SRC = os.path.join(HERE, "tools_src", "launch_count.cpp")
LC_LIB = os.path.join(HERE, "liblaunchcount.so")


def build_launch_counter():
    """CUPTI kernel counter used by bench.py for gpu_launches (measurement only)."""
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    inc = os.path.join(cuda, "targets", "x86_64-linux", "include")
    lib = os.path.join(cuda, "targets", "x86_64-linux", "lib")
    if not os.path.exists(os.path.join(inc, "cupti.h")):
        return None
    cmd = ["g++", "-O2", "-shared", "-fPIC", "-std=c++17", "-I", inc, LC_SRC, "-o", LC_LIB, "-L", lib, "-lcupti",
           f"-Wl,-rpath,{lib}"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("launch counter build failed:\n" + out.stdout + out.stderr)
    return LC_LIB


def _drain(procs):
    errs = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            errs.append(f"{src}:\n{out.decode()}")
    procs.clear()
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
