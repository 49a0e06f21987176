"""Time the Kronecker-apply GEMMs (ours, DMMA) against cuBLAS DGEMM (torch) and
the R(A) product, on one GPU.  Usage: python tools/gemm_bench.py [n] [k]"""

import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_00233_b200 as kb  # noqa: E402
from paper_2410_00233_b200 import _lib, device as D  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    lib = _lib.load()
    dev = torch.device("cuda")
    x = torch.randn(n, n, dtype=torch.float64, device=dev)
    g = torch.randn(k, n, n, dtype=torch.float64, device=dev)
    f = torch.randn(k, n, n, dtype=torch.float64, device=dev)
    tmp = torch.empty(k, n, n, dtype=torch.float64, device=dev)
    y = torch.empty(n, n, dtype=torch.float64, device=dev)
    st = D.stream_ptr()
    flops = 2.0 * k * n ** 3

    def ours_stage1():
        lib.kb_dgemm(0, 0, n, n, n, x.data_ptr(), n, 0, 0, g.data_ptr(), n, n * n, 0, tmp.data_ptr(), n, n * n,
                     k, 1, 0.0, st)

    def ours_stage2():
        lib.kb_dgemm(1, 0, n, n, n, f.data_ptr(), n, 0, n * n, tmp.data_ptr(), n, 0, n * n, y.data_ptr(), n, 0,
                     1, k, 0.0, st)

    def cublas_stage1():
        torch.matmul(x.unsqueeze(0), g, out=tmp)

    ft = f.transpose(1, 2)

    def cublas_stage2():
        # sum_i F_i^T P_i as one GEMM with inner dim k*n
        torch.mm(ft.permute(1, 0, 2).reshape(n, k * n), tmp.reshape(k * n, n), out=y)

    for name, fn in [("ours stage1 (batched)", ours_stage1), ("ours stage2 (seg-reduce)", ours_stage2),
                     ("cuBLAS stage1", cublas_stage1), ("cuBLAS stage2", cublas_stage2)]:
        t = timeit(fn)
        print(f"{name:28s} {t * 1e3:8.3f} ms  {flops / t / 1e12:6.2f} TFLOP/s")

    # the real Kronecker apply (both stages, split-K on the reduced stage)
    fk = f.reshape(k, n * n).contiguous()
    gk = g.reshape(k, n * n).contiguous()
    kr = _lib.KbKron(n, n, n, n, k, fk.data_ptr(), gk.data_ptr())
    nb = C.c_size_t()
    lib.kb_kron_workspace_bytes(C.byref(kr), C.byref(nb))
    wsb = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    xv = torch.randn(n * n, dtype=torch.float64, device=dev)
    yv = torch.empty(n * n, dtype=torch.float64, device=dev)
    for tr in (0, 1):
        t = timeit(lambda: lib.kb_kron_apply(C.byref(kr), xv.data_ptr(), yv.data_ptr(), tr, wsb.data_ptr(),
                                              nb.value, st))
        print(f"kron_apply transpose={tr}       {t * 1e3:8.3f} ms  {2 * flops / t / 1e12:6.2f} TFLOP/s")

    # correctness spot check of ours vs torch
    ours_stage1()
    ref = torch.matmul(x.unsqueeze(0), g)
    print("stage1 max err", (tmp - ref).abs().max().item())

    # R(A) product
    from paper_2410_00233_b200 import datagen

    psf = datagen.mixture_psf(n)
    op = kb.RearrangedBlur(psf, n)
    q = torch.randn(n * n, dtype=torch.float32, device=dev)
    t = timeit(lambda: op.matvec(q), reps=50)
    bmv = 4 * (2 * n * n + (n + 1) ** 2)
    print(f"R(A) matvec standalone {t * 1e6:8.1f} us  {bmv / t / 1e9:8.1f} GB/s (includes python overhead)")


if __name__ == "__main__":
    main()
