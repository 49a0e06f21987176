"""Pinned / pageable H2D bandwidth and the e2e PSF scan/upload pieces on this box."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
from paper_2410_00233_b200 import _lib, datagen, device as D
import paper_2410_00233_b200 as kb
for mb in (4, 8, 16):
    n = mb << 20
    pin = torch.empty(n, dtype=torch.uint8, pin_memory=True); dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    pag = torch.empty(n, dtype=torch.uint8)
    for src, name in ((pin, "pinned"), (pag, "pageable")):
        dev.copy_(src, non_blocking=True); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20): dev.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 20
        print(f"{name:8s} {mb:3d} MB: {dt*1e6:8.1f} us  {n/dt/1e9:6.1f} GB/s")
lib = _lib.load()
psf = datagen.make_problem("n1024").psf
s, m = C.c_double(), C.c_double()
for th in (4, 8, 16):
    lib.kb_psf_scan(psf.ctypes.data, psf.size, th, C.byref(s), C.byref(m))
    t = time.perf_counter()
    for _ in range(20): lib.kb_psf_scan(psf.ctypes.data, psf.size, th, C.byref(s), C.byref(m))
    print("scan threads", th, (time.perf_counter() - t) / 20 * 1e6, "us")
raw = torch.empty(psf.shape, dtype=torch.float64, device="cuda")
for th in (4, 8, 16):
    lib.kb_stage_upload(psf.ctypes.data, psf.nbytes, raw.data_ptr(), th, D.stream_ptr()); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20): lib.kb_stage_upload(psf.ctypes.data, psf.nbytes, raw.data_ptr(), th, D.stream_ptr())
    torch.cuda.synchronize()
    print("stage_upload threads", th, (time.perf_counter() - t) / 20 * 1e6, "us")
