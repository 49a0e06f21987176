import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2410_00233_b200.blurmodel import Psf
from paper_2410_00233_b200 import datagen
k = datagen.make_problem("n1024").psf
p = Psf(k)
out = torch.empty(k.shape, dtype=torch.float32, pin_memory=True)
on = out.numpy()
def tm(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e3

print("np.divide single", tm(lambda: np.divide(p._raw, p._total, out=on, casting="same_kind")))
print("pinned alloc", tm(lambda: torch.empty(k.shape, dtype=torch.float32, pin_memory=True)))
print("H2D 4MB non_blocking+sync", tm(lambda: out.to("cuda", non_blocking=True)))
print("Psf init", tm(lambda: Psf(k)))
import os; print("cpus", os.cpu_count())
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import device as D
n = 1024
def dk():
    b = kb.RearrangedBlur(k, n)
    t0 = time.perf_counter()
    b._device_kernels()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3
for _ in range(3): dk()
r = np.array([dk() for _ in range(20)])
print("device_kernels host ms", r[:, 0].mean(), "sync wait ms", r[:, 1].mean())
def dk2():
    b = kb.RearrangedBlur(k, n)
    stage = torch.empty(b.psf.shape, dtype=torch.float32, pin_memory=True)
    t0 = time.perf_counter()
    np.copyto(stage.numpy(), b.psf.kernel, casting="same_kind")
    t1 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    kd = stage.to(D.device(), non_blocking=True)
    e1.record()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, e0.elapsed_time(e1)
for _ in range(3): dk2()
r = np.array([dk2() for _ in range(20)])
print("normalise %.3f  launch-copy %.3f  sync %.3f  device-copy %.3f ms" % tuple(r.mean(0)))
raw = p._raw
def pageable():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(); d = torch.from_numpy(raw).to("cuda"); e1.record(); torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1)
for _ in range(3): pageable()
r = np.array([pageable() for _ in range(20)]); print("pageable raw fp64 8MB: wall %.3f device %.3f ms" % tuple(r.mean(0)))
def single_then_copy():
    stage = torch.empty(raw.shape, dtype=torch.float32, pin_memory=True)
    np.divide(raw, p._total, out=stage.numpy(), casting="same_kind")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); d = stage.to("cuda", non_blocking=True); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for _ in range(3): single_then_copy()
print("single-thread normalise then copy: device %.3f ms" % np.mean([single_then_copy() for _ in range(20)]))
static = torch.empty(raw.shape, dtype=torch.float32, pin_memory=True)
def rewrite_static():
    np.copyto(static.numpy(), p.kernel, casting="same_kind")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); d = static.to("cuda", non_blocking=True); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for _ in range(3): rewrite_static()
print("threaded rewrite of one static buffer then copy: device %.3f ms" % np.mean([rewrite_static() for _ in range(20)]))
