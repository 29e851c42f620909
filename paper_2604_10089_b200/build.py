"""Builds libbpqn.so in-tree for sm_100a (nvcc; no torch JIT cache involved)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbpqn.so")
SOURCES = ["capi.cu", "geometry.cu", "allpairs.cu", "layer.cu", "gmres.cu", "contacts.cu", "comm.cu", "diag.cu", "dense_lo.cu", "fmm.cu", "pqn.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "bpqn.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        o = os.path.join(objdir, s + ".o")
        cmd = [NVCC] + FLAGS + ["-c", os.path.join(CSRC, s), "-o", o]
        if s.endswith(".cpp"):
            cmd += ["-Xcompiler", "-fopenmp", "-Xcompiler", "-march=x86-64-v3"]
        if s.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(o)
    failed = False
    for s, pr in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        if pr.returncode != 0:
            failed = True
    if failed:
        raise RuntimeError("nvcc failed")
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB] + objs +
                          ["-lcudart", "-lgomp", "-ldl"])
    build_example()
    return LIB


EXAMPLE_SRC = os.path.join(HERE, "..", "examples", "bpqn_mvp.c")
EXAMPLE_BIN = os.path.join(HERE, "..", "examples", "bpqn_mvp")


def build_example():
    """examples/bpqn_mvp: a plain-C client of the C ABI (no Python), rpath to the in-tree .so."""
    if not os.path.exists(EXAMPLE_SRC):
        return None
    cuda = os.path.dirname(os.path.dirname(NVCC))
    subprocess.check_call(["gcc", "-O2", EXAMPLE_SRC, "-o", EXAMPLE_BIN, "-I" + os.path.join(cuda, "include"),
                           "-L" + HERE, "-lbpqn", "-L" + os.path.join(cuda, "lib64"), "-lcudart", "-lm",
                           "-Wl,-rpath,$ORIGIN/../paper_2604_10089_b200"])
    return EXAMPLE_BIN


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
