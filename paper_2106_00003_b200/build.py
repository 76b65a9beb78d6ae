"""Build the sm_100a C-ABI library in-tree: paper_2106_00003_b200/libgivens.so.

nvcc cross-compiles for sm_100a without a GPU. The .so is git-ignored but travels to the GPU
box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SRC = os.path.join(CSRC, "givens.cu")
RING_SRC = os.path.join(CSRC, "ring_inst.cu")
DEPS = [SRC, RING_SRC, os.path.join(CSRC, "ring.cuh"), os.path.join(CSRC, "common.cuh"),
        os.path.join(CSRC, "gemm_path.inc"), os.path.join(CSRC, "tc_gemm.cuh"),
        os.path.join(ROOT, "include", "givens.h")]
LIB = os.path.join(HERE, "libgivens.so")
OBJ = os.path.join(HERE, "build_obj")
# (W, L) ring configurations; must match GK_RING_CONFIGS in csrc/givens.cu
RING_CONFIGS = [(4, 1), (8, 1), (16, 1), (32, 1), (16, 4), (16, 8), (16, 16), (16, 32), (8, 64), (16, 64),
                (32, 32), (16, 128), (8, 32), (8, 128), (8, 16)]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-diag-suppress", "177",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit (the ring configurations in parallel) and link the .so."""
    if not (force or needs_build()):
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ, exist_ok=True)
    jobs = [([NVCC, *FLAGS, "-c", "-o", os.path.join(OBJ, "givens.o"), SRC], "givens.o")]
    for w, l in RING_CONFIGS:
        o = os.path.join(OBJ, f"ring_{w}_{l}.o")
        jobs.append(([NVCC, *FLAGS, f"-DRING_W={w}", f"-DRING_L={l}", "-c", "-o", o, RING_SRC], o))

    def run(job):
        cmd, _ = job
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, "givens.o")] + [os.path.join(OBJ, f"ring_{w}_{l}.o") for w, l in RING_CONFIGS]
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
