"""Build libmrv.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmrv.so")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("kernels.cu", "scene.cpp")]
DEPS = SRCS + [os.path.join(HERE, "csrc", f) for f in ("mrv_internal.h", "scene_impl.h")] + \
    [os.path.join(ROOT, "include", "mrv.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "static", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = [NVCC] + FLAGS + ["-o", LIB] + SRCS
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as f:
            f.write(r.stderr)
        if verbose:
            print(r.stderr)
    return LIB


EXAMPLE_SRC = os.path.join(ROOT, "examples", "mrv_example.c")
EXAMPLE = os.path.join(ROOT, "examples", "mrv_example")


def build_example(force: bool = False) -> str:
    """The plain-C consumer of the ABI (examples/mrv_example.c), linked against libmrv.so."""
    if force or not os.path.exists(EXAMPLE) or \
            os.path.getmtime(EXAMPLE) < max(os.path.getmtime(EXAMPLE_SRC), os.path.getmtime(LIB)):
        cuda = os.path.dirname(os.path.dirname(NVCC))
        cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-pedantic", EXAMPLE_SRC,
               "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(cuda, "include"),
               "-L" + HERE, "-lmrv", "-L" + os.path.join(cuda, "lib64"), "-lcudart",
               "-Wl,-rpath,$ORIGIN/../paper_2604_23960_b200", "-Wl,-rpath," + os.path.join(cuda, "lib64"),
               "-o", EXAMPLE]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("example build failed:\n" + r.stdout + r.stderr)
    return EXAMPLE


if __name__ == "__main__":
    build(force=True, verbose=True)
