"""Timing of the tiled R(A) block product (kb_op_apply / kb_op_apply_block) alone:
10 products per CUDA-graph replay, CUDA events, algorithmic bytes 4 (2 nv N + (n+1)^2)
against MEASURED_PEAKS.json.  Usage: python tools/ra_block_bench.py [n ...]"""

import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_00233_b200 as kb  # noqa: E402
from paper_2410_00233_b200 import _lib, datagen  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [1024, 2048]
    lib = _lib.load()
    hbm = peak()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for n in sizes:
        N = n * n
        psf = datagen.mixture_psf(n, seed=n + 1)
        blur = kb.RearrangedBlur(psf, n)
        ops = blur.op_struct()
        nb = C.c_size_t()
        lib.kb_op_workspace_bytes(C.byref(ops), C.byref(nb))
        ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
        for nv in [int(v) for v in os.environ.get("RA_NV", "1,4,8,16").split(",")]:
            X = torch.randn(nv, N, dtype=torch.float32, device="cuda")
            Y = torch.empty_like(X)
            st = torch.cuda.current_stream().cuda_stream
            lib.kb_op_apply_block(C.byref(ops), X.data_ptr(), N, Y.data_ptr(), N, nv, 0, ws.data_ptr(), nb.value, st)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            reps = 10
            with torch.cuda.graph(g):
                sp = torch.cuda.current_stream().cuda_stream
                for i in range(reps):
                    lib.kb_op_apply_block(C.byref(ops), X.data_ptr(), N, Y.data_ptr(), N, nv, i & 1, ws.data_ptr(),
                                          nb.value, sp)
            g.replay()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(3):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    g.replay()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e-3 / (5 * reps))
            by = 4.0 * (2 * nv * N + (n + 1) ** 2)
            print(f"n={n} nv={nv:2d}: {best * 1e6:8.2f} us  {by / best / 1e9:8.1f} GB/s  frac {by / best / 1e9 / hbm:.3f}",
                  flush=True)


if __name__ == "__main__":
    main()
