"""Host->device PSF path timing: RearrangedBlur(psf_host) (scan, normalise, upload) + sync."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
prob = datagen.make_problem("n1024")
psf = np.ascontiguousarray(prob.psf)
for _ in range(5):
    kb.RearrangedBlur(psf, prob.n).psf.device_normalised(np.float32)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    b = kb.RearrangedBlur(psf, prob.n)
    _ = b.psf.device_normalised(np.float32)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(os.environ.get("KB_STAGE_CHUNKS", "default"), "median us", np.median(ts) * 1e6, "min us", min(ts) * 1e6)

# variant: scan without a staged copy, normalise straight from the host array
import ctypes as C
from paper_2410_00233_b200 import _lib, device as D
lib = _lib.load()
out = D.empty(psf.shape, np.float32)
ts = []
for it in range(55):
    t0 = time.perf_counter()
    total, kmin = C.c_double(), C.c_double()
    _lib.check(lib.kb_psf_scan(psf.ctypes.data, psf.size, 16, C.byref(total), C.byref(kmin)))
    _lib.check(lib.kb_psf_commit_f32(psf.ctypes.data, psf.size, total.value, out.data_ptr(), 16, D.stream_ptr()))
    torch.cuda.synchronize()
    if it >= 5:
        ts.append(time.perf_counter() - t0)
want = kb.RearrangedBlur(psf, prob.n).psf.device_normalised(np.float32)
print("direct median us", np.median(ts) * 1e6, "min us", min(ts) * 1e6, "bitwise", bool(torch.equal(out, want)))
t0 = time.perf_counter(); [lib.kb_psf_scan(psf.ctypes.data, psf.size, 16, C.byref(total), C.byref(kmin)) for _ in range(50)]
print("scan only us", (time.perf_counter() - t0) / 50 * 1e6)
