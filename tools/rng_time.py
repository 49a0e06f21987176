"""Device time of kb_normal_pcg64 vs numpy's host draws."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_00233_b200.rng import standard_normal
for count in (1 << 20, 1 << 22, 262144 * 30):
    for _ in range(3):
        standard_normal(0, count, np.float32)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        standard_normal(0, count, np.float32)
    b.record(); torch.cuda.synchronize()
    t = time.perf_counter(); np.random.default_rng(0).standard_normal(count).astype(np.float32); th = time.perf_counter() - t
    print(f"count {count}: device {a.elapsed_time(b)/10*1e3:.1f} us, host numpy {th*1e3:.1f} ms")
