"""Timeline of one bench step (egkb + assemble at n=1024): kernels/memcpys with
start offsets and durations from the torch profiler (CUPTI), to see host gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
n = 1024
prob = datagen.make_problem("n1024")
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
scheme = kb.BlockScheme.square_image(n)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
keep = []
for _ in range(4):
    svd, tr = kb.egkb(blur, cfg); keep.append(kb.assemble(svd, scheme))
    keep = keep[-1:]
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
flush.zero_(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with torch.profiler.record_function("STEP"):
        svd, tr = kb.egkb(blur, cfg)
        op = kb.assemble(svd, scheme)
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
step = [e for e in prof.events() if e.name == "STEP"][0]
t0 = step.time_range.start
print("STEP host span us", step.time_range.end - step.time_range.start)
for e in sorted(ev, key=lambda e: e.time_range.start):
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:90]}")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith(("cuda", "aten"))]
for e in sorted(cpu, key=lambda e: e.time_range.start)[:60]:
    print(f"   cpu {e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:60]}")
