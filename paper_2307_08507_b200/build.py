"""Build the in-tree CUDA library (sm_100a) with nvcc: libmdot_b200.so.

Kept in-tree (not pip-installed) so the .so travels to the GPU box with the
repo snapshot and the driver sees it loaded from the repo."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", f) for f in ("kernels.cu", "eval_tma.cu", "persist.cu", "batch.cu", "round.cu", "solver.cu", "comm.cu", "screen.cu")]
HDR = [os.path.join(HERE, "csrc", f) for f in ("internal.cuh", "solver.h", "comm.h", "ops.cuh", "k1_tma.cuh", "entry.cuh", "umma.cuh")] + \
      [os.path.join(ROOT, "include", "mdot.h")]
OUT = os.path.join(HERE, "libmdot_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "--expt-relaxed-constexpr",
         "-shared", "-cudart", "static", "-ldl"]


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(f) > t for f in SRC + HDR)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    cmd = [NVCC] + FLAGS + ["-o", OUT + ".tmp"] + SRC
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(OUT + ".tmp", OUT)
    return OUT


CHECKED = os.path.join(ROOT, "build", "libchecked.so")


def build_checked(force=False, verbose=False):
    """The MDOT_CHECKED variant (device bounds traps + workspace guard bands),
    loaded by tests/test_gpu_checked.py through MDOT_LIB."""
    if not force and os.path.exists(CHECKED) and all(os.path.getmtime(f) <= os.path.getmtime(CHECKED)
                                                      for f in SRC + HDR):
        return CHECKED
    os.makedirs(os.path.dirname(CHECKED), exist_ok=True)
    cmd = [NVCC] + FLAGS + ["-DMDOT_CHECKED", "-o", CHECKED + ".tmp"] + SRC
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(CHECKED + ".tmp", CHECKED)
    return CHECKED


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
