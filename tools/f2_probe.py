"""Probe for SURVEY §8(f2): GEMM options for Y = U X at C3 (n=1024, m=65536): SGEMM (IEEE fp32),
TF32, and cuBLAS's BF16x9 FP32 emulation (via ctypes on the cuBLAS torch loaded). Prints time and
relative error vs an fp64 reference on a column sample."""
import ctypes
import glob
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

n, m = 1024, 65536
dev = "cuda"
U = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64))[0].float().to(dev)
X = torch.from_numpy(synth.normal_matrix(n, m, 1, synth.TID_X)).to(dev)
ref = (U.double()[:, :] @ X[:, :512].double())


def timeit(f, reps=10):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def err(Y):
    return float(torch.linalg.norm(Y[:, :512].double() - ref) / torch.linalg.norm(ref))


for prec in ["ieee", "tf32"]:
    torch.backends.cuda.matmul.fp32_precision = prec
    Y = U @ X
    t = timeit(lambda: torch.matmul(U, X, out=Y))
    print(f"torch matmul {prec}: {t:.3f} ms  {2*n*n*m/t/1e9:.1f} TF/s  rel err {err(Y):.2e}", flush=True)
    G = torch.from_numpy(synth.normal_matrix(n, m, 2, synth.TID_DY)).to(dev)
    t = timeit(lambda: G @ X.T)
    print(f"  Gamma = dY X^T {prec}: {t:.3f} ms", flush=True)
torch.backends.cuda.matmul.fp32_precision = "ieee"

libs = [l for l in open("/proc/self/maps").read().split() if "libcublas.so" in l and "Lt" not in l]
path = sorted(set(libs))[0]
print("cublas:", path)
cb = ctypes.CDLL(path)
h = ctypes.c_void_p()
print("create", cb.cublasCreate_v2(ctypes.byref(h)))
ver = ctypes.c_int()
cb.cublasGetVersion_v2(h, ctypes.byref(ver))
print("version", ver.value)
cb.cublasSetStream_v2(h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
print("setws", cb.cublasSetWorkspace_v2(h, ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel())))
alpha, beta = ctypes.c_float(1.0), ctypes.c_float(0.0)
Y = torch.empty(n, m, device=dev)
CUDA_R_32F = 0
for ct, name in [(68, "32F"), (78, "32F_EMULATED_16BFX9"), (77, "32F_FAST_TF32")]:
    def f():
        return cb.cublasGemmEx(h, 0, 0, m, n, n, ctypes.byref(alpha), ctypes.c_void_p(X.data_ptr()), CUDA_R_32F, m,
                               ctypes.c_void_p(U.data_ptr()), CUDA_R_32F, n, ctypes.byref(beta),
                               ctypes.c_void_p(Y.data_ptr()), CUDA_R_32F, m, ct, -1)
    rc = f()
    torch.cuda.synchronize()
    if rc != 0:
        print(name, "rc", rc)
        continue
    t = timeit(f)
    print(f"cublasGemmEx {name}: {t:.3f} ms  {2*n*n*m/t/1e9:.1f} TF/s  rel err {err(Y):.2e}", flush=True)
# math-mode route
print("mathmode", cb.cublasSetMathMode(h, 4))
rc = cb.cublasGemmEx(h, 0, 0, m, n, n, ctypes.byref(alpha), ctypes.c_void_p(X.data_ptr()), CUDA_R_32F, m,
                     ctypes.c_void_p(U.data_ptr()), CUDA_R_32F, n, ctypes.byref(beta),
                     ctypes.c_void_p(Y.data_ptr()), CUDA_R_32F, m, 68, -1)
torch.cuda.synchronize()
print("emul via math mode rc", rc, "err", err(Y))
