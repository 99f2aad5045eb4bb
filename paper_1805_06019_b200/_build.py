"""Build the native libraries in-tree (sm_100a CUDA + C++ producer).

Built artefacts land next to the sources (git-ignored, shipped to the GPU box
with the snapshot): paper_1805_06019_b200/librlfc_b200.so and
paper_1805_06019_b200/librlfc_producer.so.
"""

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
PRODUCER = os.path.join(PKG, "producer")
ROOT = os.path.dirname(PKG)

CUDA_LIB = os.path.join(PKG, "librlfc_b200.so")
PRODUCER_LIB = os.path.join(PKG, "librlfc_producer.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
              "-shared", "-I" + os.path.join(ROOT, "include")]


def _newer(target, sources):
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(s) <= t for s in sources)


def _sources(d, exts):
    return sorted(os.path.join(d, f) for f in os.listdir(d)
                  if os.path.splitext(f)[1] in exts)


def build_cuda(force=False, verbose=False):
    cus = _sources(CSRC, {".cu"})
    deps = cus + _sources(CSRC, {".cuh", ".h"}) + [
        os.path.join(ROOT, "include", "rlfc_b200.h")]
    if not force and _newer(CUDA_LIB, deps):
        return CUDA_LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc] + NVCC_FLAGS + ["-o", CUDA_LIB] + cus
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return CUDA_LIB


def build_producer(force=False, verbose=False):
    srcs = _sources(PRODUCER, {".cpp"})
    deps = srcs + _sources(PRODUCER, {".h", ".hpp"})
    if not srcs:
        return None
    if not force and _newer(PRODUCER_LIB, deps):
        return PRODUCER_LIB
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
           "-ffp-contract=off", "-fno-fast-math", "-o", PRODUCER_LIB] + srcs
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return PRODUCER_LIB


def build_all(force=False, verbose=False):
    build_cuda(force, verbose)
    build_producer(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
