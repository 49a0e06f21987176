"""Time the fused eGKB (fast engine) at configs[3] (n=1024) and configs[4] (n=2048):
median of 10 calls with the L2 flushed before each, plus the rank decision and the
leading singular values.  Usage: python tools/egkb_time.py [config ...]"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_00233_b200 as kb  # noqa: E402
from paper_2410_00233_b200 import datagen  # noqa: E402


def main():
    names = sys.argv[1:] or ["n1024", "n2048"]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name in names:
        prob = datagen.make_problem(name)
        blur = kb.RearrangedBlur(prob.psf, prob.n)
        cfg = kb.EgkbConfig(**prob.egkb)
        for _ in range(3):
            svd, tr = kb.egkb(blur, cfg)
        ts = []
        for _ in range(10):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            svd, tr = kb.egkb(blur, cfg)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        sig = np.asarray(svd.sigma)
        import hashlib
        hv = hashlib.sha1(np.asarray(tr.alphas + tr.ts, np.float64).tobytes() + sig.tobytes()
                          + np.ascontiguousarray(svd.v[:, :2]).tobytes()).hexdigest()[:12]
        print(f"{name}: median {np.median(ts):.3f} ms  min {min(ts):.3f} ms  chosen_k={tr.chosen_k} k_p={tr.k_p} "
              f"stop={tr.stop_reason} breakdown={tr.breakdown} sigma[:4]={sig[:4]} hash={hv}", flush=True)


if __name__ == "__main__":
    main()
