"""Benchmark of the hot path on BASELINE.json configs[3] (n=1024).

One STEP = one Kronecker-product approximation of the n=1024 blur: fp32 eGKB
on the matrix-free R(A) with the config's "rank 30 + enlargement p=2"
(EgkbConfig(k_max=30, k_min=30, p=2, tau=1e300); the fp32 recurrence breaks
down at the numerical rank, as the reference does) followed by `assemble`
into fp64 Kronecker factors.  `value` = approximations/s over all ranks with
inputs resident in HBM; `e2e` = the same through the public API from host
arrays (PSF uploaded, the reference's y0 stream drawn on the device by kb_rng.cu, trace/sigma read back) each
step.  The same run also measures the fp64 split-Bregman solve that consumes
the factors (isotropic, 200 outer iterations, CGLS i_max=100 tau=1e-4: the
north star's approximation + solve, "n1" and "sb"), the reference-arithmetic
engine ("reference_arithmetic"), and the R(A) product ("ra_matvec").

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU (torchrun): independent replicas (weak scaling), max-over-ranks time.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "n1024"
FP64_PEAK_TFLOPS = 37.2   # DMMA m8n8k4 issue rate measured on this pool (profiles/fp64_peak_r01.txt)
METRIC = "R(A) matvec GB/s & KP-approx time at n=1024; SB iter/s; % of roofline"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def egkb_cfg_kwargs():
    from paper_2410_00233_b200 import datagen

    return dict(datagen.CONFIGS[CONFIG]["egkb"])


def bench_config(n):
    """The workload, identical in both arms' JSON lines (results live under "result")."""
    return {"workload": "configs[3] n=1024 fp32 eGKB rank 30+2 (matrix-free R(A)) -> assemble", "n": n,
            "egkb": {k: (str(v) if k == "tau" else v) for k, v in egkb_cfg_kwargs().items()},
            "l2": "GPU arm: flushed (512 MB write) before every timed step"}


def trace_result(tr):
    return {"chosen_k": int(tr.chosen_k), "k_p": int(tr.k_p), "stop_reason": str(tr.stop_reason),
            "breakdown": bool(tr.breakdown)}


def psf_f32(psf):
    """The fp32 kernel the reference's Psf + cast produce: (k / k.sum()).astype(float32)."""
    return (psf / psf.sum()).astype(np.float32)


# ---------------------------------------------------------------- clocks
class Clocks:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # nvidia-smi's first query (NVML start-up) stalls the driver for several ms:
        # let it happen before any timed work
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 5.0:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ra_block_time(kb, lib, D, n, nv, flush, hbm):
    """One nv-vector R(A) block product at side n (configs[4]'s PSF family): 10 products per
    CUDA-graph replay, 5 replays, CUDA events; algorithmic bytes 4 (2 nv N + (n+1)^2)."""
    import ctypes as C

    import torch

    from paper_2410_00233_b200 import datagen

    N = n * n
    blur = kb.RearrangedBlur(datagen.mixture_psf(n, sig_hi=12.0 if n >= 2048 else 6.0), n)
    ops = blur.op_struct()
    nb = C.c_size_t()
    lib.kb_op_workspace_bytes(C.byref(ops), C.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device=D.device())
    X = torch.randn(nv, N, dtype=torch.float32, device=D.device())
    Y = torch.empty_like(X)
    lib.kb_op_apply_block(C.byref(ops), X.data_ptr(), N, Y.data_ptr(), N, nv, 0, ws.data_ptr(), nb.value,
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        sp = torch.cuda.current_stream().cuda_stream
        for i in range(10):
            lib.kb_op_apply_block(C.byref(ops), X.data_ptr(), N, Y.data_ptr(), N, nv, i & 1, ws.data_ptr(), nb.value, sp)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_()
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / 50
    by = 4.0 * (2 * nv * N + (n + 1) ** 2)
    return {"us_per_launch": t * 1e6, "GBps": by / t / 1e9, "frac": by / t / 1e9 / hbm, "vectors": nv, "n": n}


# ---------------------------------------------------------------- reference arm
def run_reference(args, prob):
    """The reference's algorithm on the host CPU (oracle port; the reference is
    pure Python and cannot be installed on the GPU box)."""
    from types import SimpleNamespace

    from oracle import lowrank as olr
    from oracle import structured as ost

    n = prob.n
    k32 = psf_f32(prob.psf)
    cfg = SimpleNamespace(reorth=None, seed=0, break_tol=None, keep_basis=False, **egkb_cfg_kwargs())
    cfg.tau = float(cfg.tau)

    def step():
        (u, s, v), tr = olr.egkb(lambda q: ost.ra_matvec(k32, n, q), lambda x: ost.ra_rmatvec(k32, n, x),
                                 (n * n, n * n), np.float32, cfg)
        # assemble: fp64 factors sigma_i u_i, v_i (kronop.py:103-123)
        _ = [s[i].astype(np.float64) * u[:, i].astype(np.float64) for i in range(u.shape[1])]
        _ = [v[:, i].astype(np.float64) for i in range(v.shape[1])]
        return tr

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tr = step()
    dt = (time.perf_counter() - t0) / args.steps
    cores = os.cpu_count()
    val = 1.0 / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "KP-approx/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(n), "result": trace_result(tr),
        "cpu_baseline": {"value": val, "unit": "KP-approx/s", "cores": cores, "kind": "port",
                         "sample": "full eGKB+assemble per step (oracle/lowrank.py restatement of lowrank.py:159-329 "
                                   "on the numpy structured R(A), MGS as the reference)"},
        "e2e": {"value": val, "unit": "KP-approx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------- our arm
def prof_read(lib, cls):
    import ctypes as C

    ms, n, by, fl = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
    lib.kb_prof_query(cls, C.byref(ms), C.byref(n), C.byref(by), C.byref(fl))
    return ms.value, n.value, by.value, fl.value


def sweep_bench(kb, D):
    """Batched lambda sweep (splitbregman.py:195-235) at configs[0]
    (n=64): 100 log-spaced lambdas x 5 outer sweeps, CGLS(100, 1e-4), on the
    eGKB factors, against one sb_run per lambda (same kernels, unbatched)."""
    import torch

    from paper_2410_00233_b200 import datagen

    prob = datagen.make_problem("n64")
    svd, _ = kb.egkb(kb.RearrangedBlur(prob.psf, prob.n), kb.EgkbConfig(**prob.egkb))
    op = kb.assemble(svd, kb.BlockScheme.square_image(prob.n))
    gamma = datagen.LAM ** 2 / datagen.BETA
    kw = dict(gamma=gamma, lam_lo=0.01, lam_hi=1.0, count=100, x_true=prob.x_true, l_max=5, tau=0.0,
              cgls=kb.CglsConfig(100, 1e-4))
    kb.sweep(op, prob.b, **dict(kw, count=2))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    recs = kb.sweep(op, prob.b, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms_b = e0.elapsed_time(e1)
    cfgs = [kb.SbConfig.from_gamma(float(l), gamma, l_max=5, tau=0.0, cgls=kw["cgls"])
            for l in kb.lambda_grid(0.01, 1.0, 100)]
    e0.record()
    seq = [kb.sb_run(op, prob.b, c, x_true=prob.x_true) for c in cfgs]
    e1.record()
    torch.cuda.synchronize()
    ms_s = e0.elapsed_time(e1)
    its = sum(r["iota_total"] for r in recs)
    return {"config": "configs[0] n=64, k=%d: 100 lambdas (0.01..1, gamma=lam^2/beta fixed) x 5 outer, "
                      "CGLS(100, 1e-4)" % op.k,
            "batched_ms": ms_b, "sequential_ms": ms_s, "speedup": ms_s / ms_b, "cgls_iters": its,
            "cgls_it_per_s": its / (ms_b * 1e-3), "sequential_cgls_iters": sum(r.iota_total for r in seq),
            "kernel": "kb_sb_run_batch (stacked DMMA GEMMs, one launch per pass over all lambdas)"}


def other_configs(kb, D, flush):
    """configs[2] (n=512, fixed 20+2) and configs[4] (n=2048, automatic rank, cap 50): one
    approximation per engine (fast and reference arithmetic), device time with the PSF
    resident and L2 flushed, plus one CGLS iteration rate on the fast engine's factors
    (configs[2]: both SB variants; configs[4]: anisotropic)."""
    import torch

    from paper_2410_00233_b200 import datagen

    out = {}
    for name in ("n512", "n2048"):
        prob = datagen.make_problem(name)
        blur = kb.RearrangedBlur(prob.psf, prob.n)
        cfg = kb.EgkbConfig(**prob.egkb)
        rec = {"n": prob.n, "egkb": {k: (str(v) if k == "tau" else v) for k, v in prob.egkb.items()}}
        for arith in ("fast", kb.host_blas_arithmetic()):
            for _ in range(2):   # warm-up: allocator, kernel attributes, two live result sets
                svd, tr = kb.egkb(blur, cfg, arithmetic=arith)
                op = kb.assemble(svd, kb.BlockScheme.square_image(prob.n))
            ms = []
            for _ in range(5):
                flush.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                svd, tr = kb.egkb(blur, cfg, arithmetic=arith)
                op = kb.assemble(svd, kb.BlockScheme.square_image(prob.n))
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            rec["fast" if arith == "fast" else "reference_arithmetic"] = {
                "ms": float(np.median(ms)), "ms_min": float(min(ms)), "result": trace_result(tr)}
            if arith == "fast":
                fop = op
        if name == "n512":   # configs[2]'s other engines: TSVD-20 and RSVD (k=20, p=10, q=2)
            def dev_ms(fn, reps=3):
                fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                return e0.elapsed_time(e1) / reps
            rec["tsvd20_ms"] = dev_ms(lambda: kb.tsvd(blur, 20))
            try:
                kb.rsvd(blur, kb.RsvdConfig(k=20, p=10, q=2, seed=0))
                rec["rsvd_20_10_2"] = "ok"
            except kb.RankDeficiencyError as e:
                rec["rsvd_20_10_2"] = f"RankDeficiencyError(column {e.column}) (the reference raises the same)"
            for k in range(6, 1, -1):   # the largest fp32 block (p = 2) the random draw keeps full rank
                try:
                    kb.rsvd(blur, kb.RsvdConfig(k=k, p=2, q=2, seed=0))
                except kb.RankDeficiencyError:
                    continue
                rec[f"rsvd_{k}_2_2_ms"] = dev_ms(lambda: kb.rsvd(blur, kb.RsvdConfig(k=k, p=2, q=2, seed=0)))
                rec["rsvd_note"] = f"k={k}, p=2, q=2: the largest k with p=2 that passes the rank check"
                break
        variants = ["isotropic", "anisotropic"] if name == "n512" else ["anisotropic"]
        b_dev = D.to_device(prob.b)
        for var in variants:
            c = kb.SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant=var, tau=0.0, l_max=1,
                            cgls=kb.CglsConfig(i_max=100, tau=1e-4))
            kb.sb_run(fop, b_dev, c)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = kb.sb_run(fop, b_dev, c)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            rec[f"sb_{var}"] = {"k_terms": fop.k, "outer_it_ms": t, "cgls_iters": int(sum(r.cgls_iters)),
                                "cgls_it_per_s": sum(r.cgls_iters) / (t * 1e-3)}
            try:   # the same sweep on the operator's Toeplitz split (opt-in, see n1.toeplitz_split)
                sp, dropped = fop.toeplitz_split()
                kb.sb_run(sp, b_dev, c)
                torch.cuda.synchronize()
                e0.record()
                r2 = kb.sb_run(sp, b_dev, c)
                e1.record()
                torch.cuda.synchronize()
                t2 = e0.elapsed_time(e1)
                rec[f"sb_{var}"]["toeplitz_split"] = {
                    "outer_it_ms": t2, "cgls_iters": int(sum(r2.cgls_iters)),
                    "cgls_it_per_s": sum(r2.cgls_iters) / (t2 * 1e-3), "dropped_rel_frobenius": dropped}
                del sp, r2
            except Exception as exc:   # noqa: BLE001
                rec[f"sb_{var}"]["toeplitz_split"] = {"error": f"{type(exc).__name__}: {exc}"}
        out[name] = rec
    return out


def egkb_alg_bytes(n, kh, kw, k_p, k):
    """B_egkb = (2k_p+1) B_mv + sum_{j=1..k_p} 8N(2j+3) + 4N(2k_p+1+2k),
    B_mv = 4 (2N + kh kw) (K counted once per product)."""
    N = n * n
    bmv = 4.0 * (2 * N + kh * kw)
    return (2 * k_p + 1) * bmv + sum(8.0 * N * (2 * j + 3) for j in range(1, k_p + 1)) + 4.0 * N * (2 * k_p + 1 + 2 * k)


def sharded_bench(kb, D, world, dist, peak):
    """configs[4] (n=2048, automatic rank, cap 50) and configs[3] (n=1024, 30+2) with the
    Krylov vectors row-sharded over all ranks (parallel.sharded_egkb: three int64 limb
    allreduces per half step over NCCL).  Device time, max over ranks; the result is
    identical for any number of ranks.  Whole-box roofline: the run's algorithmic bytes
     over ranks x the HBM peak.  The single-GPU fused engine on the same
    problem is timed beside it (rank 0's device)."""
    import torch

    from paper_2410_00233_b200 import datagen
    from paper_2410_00233_b200.parallel import sharded_egkb

    def timed(fn, reps=3):
        ms = []
        for _ in range(reps):
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = torch.tensor([float(np.median(ms))], dtype=torch.float64, device=D.device())
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    res = {}
    for name, label in (("n2048", "configs[4] n=2048, EgkbConfig(k_max=50)"),
                        ("n1024", "configs[3] n=1024, EgkbConfig(30, k_min=30, p=2, tau=1e300)")):
        prob = datagen.make_problem(name)
        blur = kb.RearrangedBlur(prob.psf, prob.n)
        cfg = kb.EgkbConfig(**prob.egkb)
        for _ in range(2):
            sharded_egkb(blur, cfg)
        ms, (svd, tr) = timed(lambda: sharded_egkb(blur, cfg))
        kh, kw = blur.psf.shape
        alg = egkb_alg_bytes(prob.n, kh, kw, tr.k_p, tr.chosen_k)
        for _ in range(2):
            kb.egkb(blur, cfg)
        fused_ms, _ = timed(lambda: kb.egkb(blur, cfg))
        res[name] = {"config": label, "ranks": world, "ms": ms, "result": trace_result(tr),
                     "sigma_1": float(svd.sigma[0]),
                     "roofline_whole_box": {"alg_bytes": alg, "achieved_GBps": alg / ms * 1e-6,
                                            "peak_GBps": world * peak, "frac": alg / ms * 1e-6 / (world * peak)},
                     "fused_single_gpu_ms": fused_ms}
    res["note"] = ("rows of every Krylov vector sharded over the ranks; host loop in Python, one CUDA graph "
                   "per half step, 3 int64 allreduces per half step; bit-identical result for any rank count")
    return res


def run_ours(args, prob, rank, world, dist):
    import torch

    import paper_2410_00233_b200 as kb
    from paper_2410_00233_b200 import _lib
    from paper_2410_00233_b200 import device as D

    lib = _lib.load()
    n = prob.n
    N = n * n
    cfg = kb.EgkbConfig(**egkb_cfg_kwargs())
    scheme = kb.BlockScheme.square_image(n)
    blur = kb.RearrangedBlur(prob.psf, n)          # PSF resident on the device
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=D.device())

    def barrier():
        if dist is not None:
            dist.barrier()

    def step_resident():
        svd, tr = kb.egkb(blur, cfg)               # start vector drawn on the device (kb_rng.cu)
        op = kb.assemble(svd, scheme)
        return svd, tr, op

    # the clock sampler starts before the warm-up so its start-up is outside the timed region
    clocks = Clocks(torch.cuda.current_device()) if rank == 0 and not os.environ.get("KB_BENCH_NO_CLOCKS") else None
    # warm-up exactly like the timed loop (the previous step's results stay alive
    # while the next step allocates), so the caching allocator holds both sets
    for _ in range(max(args.warmup, 3)):
        svd, tr, op = step_resident()
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs), L2 flushed between steps.  Python's
    # cyclic GC is collected up front and paused while timing (as timeit does):
    # a collection inside a step would stall the host between the step's launches.
    gc.collect()
    gc.disable()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        ev[i][0].record()
        svd, tr, op = step_resident()
        ev[i][1].record()
        torch.cuda.synchronize()
    gc.enable()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t_max = torch.tensor([total_ms], dtype=torch.float64, device=D.device())
    if dist is not None:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total_ms = float(t_max.item())
    ms_per_step = total_ms / args.steps
    value = world * args.steps / (total_ms * 1e-3)

    # ---- profiled replay: same kernels launched eagerly, CUDA events around each
    # launch on the launching stream (per-kernel device time for the roofline)
    lib.kb_prof_enable(1)
    prof_ms = 0.0
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step_resident()
        b.record()
        torch.cuda.synchronize()
        prof_ms += a.elapsed_time(b)
    prof = {c: prof_read(lib, c) for c in range(7)}
    lib.kb_prof_enable(0)
    gpu_launches = sum(v[1] for v in prof.values())

    # ---- e2e: public API from host arrays, every step
    psf_host = prob.psf
    h2d = psf_host.size * 4                                     # K normalised + cast on the host threads, fp32 on the wire
    e2e_ms = []
    gc.collect()
    gc.disable()
    for i in range(max(args.warmup, 3) + max(args.steps, 1)):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        blur_i = kb.RearrangedBlur(psf_host, n)                 # validates + normalises the PSF, uploads K
        svd_i, tr_i = kb.egkb(blur_i, cfg)                      # reference RNG stream, drawn on the device
        op_i = kb.assemble(svd_i, scheme)
        sig = np.asarray(svd_i.sigma)                           # result on the host
        torch.cuda.synchronize()
        if i >= max(args.warmup, 3):               # the first W calls are the e2e warm-up
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    gc.enable()
    iters = len(tr.alphas) + 1
    d2h = 8 * 4 * iters + 16 + sig.nbytes
    rows_c = tr.k_p + (1 if tr.breakdown and len(tr.ts) > tr.k_p else 0)
    h2d += 4 * (rows_c + tr.k_p) * tr.chosen_k + 8 * tr.chosen_k   # lift weights + sigma (from the host SVD of C)
    e2e_t = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=D.device())
    if dist is not None:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world / (float(e2e_t.item()) * 1e-3)
    # e2e with the factors returned to host memory in the reference's layout
    # (kronop.py:42-43: k C-ordered fp64 n x n arrays per side) -- 2 k n^2 x 8 bytes more
    e2e_host_ms = []
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blur_i = kb.RearrangedBlur(psf_host, n)
        svd_i, tr_i = kb.egkb(blur_i, cfg)
        op_i = kb.assemble(svd_i, scheme)
        ax_h, ay_h = op_i.ax, op_i.ay
        e2e_host_ms.append((time.perf_counter() - t0) * 1e3)
        del ax_h, ay_h
    host_fac_bytes = 2 * 8 * op_i.k * N

    # ---- the reference-arithmetic engine (arithmetic="reference": the reference's own fp32
    # operations -- OpenBLAS sdot of this host's numpy, sequential MGS): bit-identical
    # trace and rank decision to the reference (tests/test_gpu_refarith.py)
    ref_arith = kb.host_blas_arithmetic()
    kb.egkb(blur, cfg, arithmetic=ref_arith)
    torch.cuda.synchronize()
    ra_ms = []
    for i in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0_.record()
        svd_r, tr_r = kb.egkb(blur, cfg, arithmetic=ref_arith)
        kb.assemble(svd_r, scheme)
        e1_.record()
        torch.cuda.synchronize()
        ra_ms.append(e0_.elapsed_time(e1_))
    ref_arith_line = {"engine": f"egkb(arithmetic='reference') -> {ref_arith}", "ms_per_step": float(np.mean(ra_ms)),
                      "value": world * 1e3 / float(np.mean(ra_ms)), "unit": "KP-approx/s",
                      "result": trace_result(tr_r),
                      "note": "trace, rank decision and Krylov bases bit-identical to the reference's fp32 run "
                              "on this host's OpenBLAS sdot kernel; latency-bound by construction (each MGS "
                              "coefficient is a sequential fp32 FMA chain of N/64 elements)"}

    # ---- standalone R(A) product (kb_op_apply): 50 products per CUDA-graph replay
    import ctypes as C

    q_d = torch.randn(N, dtype=torch.float32, device=D.device())
    y_d = torch.empty_like(q_d)
    ops = blur.op_struct()
    nb = C.c_size_t()
    lib.kb_op_workspace_bytes(C.byref(ops), C.byref(nb))
    mv_ws = torch.zeros(nb.value, dtype=torch.uint8, device=D.device())
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for tr_ in (0, 1):
            lib.kb_op_apply(C.byref(ops), q_d.data_ptr(), y_d.data_ptr(), tr_, mv_ws.data_ptr(), nb.value,
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.current_stream().wait_stream(side)
    mv_graph = torch.cuda.CUDAGraph()
    n_mv = 50
    with torch.cuda.graph(mv_graph):
        st_ptr = torch.cuda.current_stream().cuda_stream
        for i_ in range(n_mv):
            lib.kb_op_apply(C.byref(ops), q_d.data_ptr(), y_d.data_ptr(), i_ & 1, mv_ws.data_ptr(), nb.value, st_ptr)
    mv_graph.replay()
    torch.cuda.synchronize()
    mv_e0, mv_e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_()
    mv_e0.record()
    for _ in range(5):
        mv_graph.replay()
    mv_e1.record()
    torch.cuda.synchronize()
    mv_t = mv_e0.elapsed_time(mv_e1) * 1e-3 / (5 * n_mv)
    # block product (16 vectors per launch: the RSVD block products)
    nvb = 16
    Xb = torch.randn(nvb, N, dtype=torch.float32, device=D.device())
    Yb = torch.empty_like(Xb)
    blk_graph = torch.cuda.CUDAGraph()
    lib.kb_op_apply_block(C.byref(ops), Xb.data_ptr(), N, Yb.data_ptr(), N, nvb, 0, mv_ws.data_ptr(), nb.value,
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    with torch.cuda.graph(blk_graph):
        st_ptr = torch.cuda.current_stream().cuda_stream
        for i_ in range(10):
            lib.kb_op_apply_block(C.byref(ops), Xb.data_ptr(), N, Yb.data_ptr(), N, nvb, i_ & 1, mv_ws.data_ptr(),
                                  nb.value, st_ptr)
    blk_graph.replay()
    torch.cuda.synchronize()
    flush.zero_()
    mv_e0.record()
    for _ in range(5):
        blk_graph.replay()
    mv_e1.record()
    torch.cuda.synchronize()
    blk_t = mv_e0.elapsed_time(mv_e1) * 1e-3 / 50

    # ---- split Bregman on the fresh factors (same run): one outer sweep
    sb_cfg = kb.SbConfig(lam=0.1150, beta=0.0066, variant="isotropic", tau=0.0, l_max=args.sb_outer,
                         cgls=kb.CglsConfig(i_max=100, tau=1e-4))
    b_dev = D.to_device(prob.b)
    sb_op = op
    if world > 1:   # Kronecker-term sharding over the ranks, one NCCL allreduce per product
        from paper_2410_00233_b200.parallel import ShardedKroneckerSum

        sb_op = ShardedKroneckerSum(op)
    kb.sb_run(sb_op, b_dev, kb.SbConfig(lam=0.1150, beta=0.0066, variant="isotropic", tau=0.0, l_max=1,
                                     cgls=kb.CglsConfig(i_max=2, tau=0.0)))   # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sb_res = kb.sb_run(sb_op, b_dev, sb_cfg)
    e1.record()
    torch.cuda.synchronize()
    sb_ms = e0.elapsed_time(e1)
    # the same solve on the operator's Toeplitz split (opt-in: one dense x banded + k banded x
    # banded terms, both GEMM stages skip all-zero tiles); single GPU only
    split_line = None
    def split_n1():
        sp_op, sp_resid = op.toeplitz_split()
        if world > 1:   # this rank's share of the banded terms, one allreduce per product
            from paper_2410_00233_b200.parallel import ShardedKroneckerSum

            sp_full = sp_op
            sp_op = ShardedKroneckerSum(sp_full)
        kb.sb_run(sp_op, b_dev, kb.SbConfig(lam=0.1150, beta=0.0066, variant="isotropic", tau=0.0, l_max=1,
                                            cgls=kb.CglsConfig(i_max=2, tau=0.0)))   # warm-up
        torch.cuda.synchronize()
        t_sp0 = time.perf_counter()
        sp_op2, _ = op.toeplitz_split()
        torch.cuda.synchronize()
        sp_split_ms = (time.perf_counter() - t_sp0) * 1e3
        e0.record()
        sp_res = kb.sb_run(sp_op, b_dev, sb_cfg)
        e1.record()
        torch.cuda.synchronize()
        sp_ms = e0.elapsed_time(e1)
        xa = sb_res.x if isinstance(sb_res.x, np.ndarray) else D.to_host(sb_res.x)
        xb = sp_res.x if isinstance(sp_res.x, np.ndarray) else D.to_host(sp_res.x)
        sp_cg = int(sum(sp_res.cgls_iters))
        split_line = {"sb_ms": sp_ms, "split_ms": sp_split_ms, "total_s": (ms_per_step + sp_split_ms + sp_ms) * 1e-3,
                      "sb_outer_iters": sp_res.outer_iters, "cgls_iters_total": sp_cg,
                      "cgls_it_per_s": sp_cg / (sp_ms * 1e-3), "terms": sp_op.k,
                      "g_band": [int(v) for v in (sp_full if world > 1 else sp_op)._band.cpu().numpy()],
                      "f_band": [int(v) for v in (sp_full if world > 1 else sp_op)._fband.cpu().numpy()],
                      "dropped_rel_frobenius": sp_resid,
                      "solution_gap_vs_dense_factors": float(np.linalg.norm(xb - xa) / np.linalg.norm(xa)),
                      "note": "KroneckerSum.toeplitz_split(): F_i = T_i + a_i D + O(rounding) for a zero-BC eGKB "
                              "approximation; an approximation of the assembled operator (not reference "
                              "arithmetic), opt-in; parity of the solve on the split operator's own factors: "
                              "tests/test_gpu_structured.py"}
        del sp_op, sp_op2, sp_res
        return split_line

    if not args.no_sweep:
        try:
            split_line = split_n1()
        except Exception as exc:   # noqa: BLE001
            split_line = {"error": f"{type(exc).__name__}: {exc}"}
    lib.kb_prof_enable(1)                      # profiled replay (one outer sweep) for the GEMM share
    sb_cfg1 = kb.SbConfig(lam=0.1150, beta=0.0066, variant="isotropic", tau=0.0, l_max=1,
                          cgls=kb.CglsConfig(i_max=100, tau=1e-4))
    e0.record()
    sb_res1 = kb.sb_run(sb_op, b_dev, sb_cfg1)
    e1.record()
    torch.cuda.synchronize()
    sb_prof_ms = e0.elapsed_time(e1)
    g_ms, g_n, g_by, g_fl = prof_read(lib, 3)
    v_ms, v_n, _, _ = prof_read(lib, 4)
    lib.kb_prof_enable(0)
    def aux(fn, *a):
        """Auxiliary sub-lines never take the headline line down with them."""
        try:
            return fn(*a)
        except Exception as exc:   # noqa: BLE001
            return {"error": f"{type(exc).__name__}: {exc}"}

    sweep = aux(sweep_bench, kb, D) if not args.no_sweep else None
    others = aux(other_configs, kb, D, flush) if not args.no_sweep else None
    sharded = aux(sharded_bench, kb, D, world, dist, peaks()[0]) if not args.no_sweep else None
    clk = clocks.stop() if clocks is not None else None
    if rank != 0:
        return

    hbm, hbm_src = peaks()
    # dominant kernel of the step: the class with the largest device time
    names = {0: "persistent eGKB (k_egkb_tiled)", 1: "R(A) products (k_rat_* tiled block product)",
             2: "R(A) K-column sums (k_colsum_seg)", 3: "fp64 GEMM (k_dgemm, DMMA)", 4: "CGLS/SB vector passes",
             5: "lift (k_lift)", 6: "start-vector draws (k_zig_*)"}
    dom = max(range(7), key=lambda c: prof[c][0])
    d_ms, d_n, d_by, d_fl = prof[dom]
    achieved = (d_by / d_n) / ((d_ms / d_n) * 1e-3) / 1e9 if d_n else 0.0
    step_share = d_ms / prof_ms if prof_ms else 0.0
    # standalone R(A) product (x read, y written, K read: SURVEY §8d B_mv)
    mv_bytes_alg = 4.0 * (2 * N + (n + 1) ** 2)
    ra = {"us_per_product": mv_t * 1e6, "GBps": mv_bytes_alg / mv_t / 1e9,
          "frac": mv_bytes_alg / mv_t / 1e9 / hbm, "bytes_per_product": mv_bytes_alg,
          "timing": f"{n_mv} products (alternating R x / R^T x) per CUDA-graph replay, 5 replays, CUDA events",
          "kernel": "k_rat_diag | k_rat_w | k_rat_z[_mma] | k_rat_bcast (TMA-streamed tile-stack diagonal sums, "
                    "fixed-order diagonal reduction, clustered row-chunk z with a DSMEM reduction, streaming "
                    "broadcast; chained by programmatic dependent launch, no grid barriers)",
          "block16": {"us_per_launch": blk_t * 1e6,
                      "GBps": 4.0 * (2 * 16 * N + (n + 1) ** 2) / blk_t / 1e9,
                      "frac": 4.0 * (2 * 16 * N + (n + 1) ** 2) / blk_t / 1e9 / hbm,
                      "note": "16 vectors per launch (RSVD block product): K read once per block"},
          "block16_n2048": aux(ra_block_time, kb, lib, D, 2048, 16, flush, hbm) if not args.no_sweep else None}
    cg = int(sum(sb_res.cgls_iters))
    # the G stage (half the dense flops of a square apply) only runs the k tiles
    # inside G's zero band (kb_kron_band); count executed DMMA flops, not dense
    band = [int(b) for b in op._band.cpu().numpy()] if getattr(op, "_band", None) is not None else None
    g_frac = 1.0
    if band is not None:
        def tile_frac(lo, hi, K=n, N=n, BN=64, BK=32):   # Cfg1 tiles, k_dgemm's band rule
            kt = 0
            for n0 in range(0, N, BN):
                klo, khi = max(0, n0 - hi), min(K - 1, n0 + BN - 1 - lo)
                kt += (khi // BK + 1 - klo // BK) if khi >= klo else 0
            return kt * BK / (K * -(-N // BN))
        g_frac = 0.5 * (tile_frac(band[0], band[1]) + tile_frac(-band[1], -band[0]))
    g_exec = g_fl * (1.0 + g_frac) / 2.0
    cg1 = int(sum(sb_res1.cgls_iters))
    sb = {"variant": "isotropic", "k_terms": op.k, "cgls": "CglsConfig(i_max=100, tau=1e-4)", "lam": 0.1150,
          "beta": 0.0066,
          "parallelism": f"Kronecker terms sharded over {world} GPU(s), NCCL allreduce per product"
          if world > 1 else "single GPU", "outer_iters": sb_res.outer_iters, "cgls_iters": cg,
          "ms": sb_ms, "outer_it_per_s": sb_res.outer_iters / (sb_ms * 1e-3),
          "cgls_it_per_s": cg / (sb_ms * 1e-3),
          "gemm_tflops": g_exec / (g_ms * 1e-3) / 1e12 if g_ms else None,
          "gemm_frac_fp64_peak": (g_exec / (g_ms * 1e-3) / 1e12) / FP64_PEAK_TFLOPS if g_ms else None,
          "gemm_dense_equiv_tflops": g_fl / (g_ms * 1e-3) / 1e12 if g_ms else None,
          "g_band": band, "g_stage_tiles_run": g_frac,
          "gemm_note": "G factors (v side) are banded Toeplitz for zero BC: the G-stage GEMM skips all-zero "
                       "k tiles (bit-identical); gemm_tflops counts executed flops",
          "gemm_share": g_ms / sb_prof_ms if sb_prof_ms else None, "vector_pass_ms": v_ms,
          "gemm_profile": f"kernel classes from a profiled replay of one outer sweep ({cg1} CGLS iterations)",
          "fp64_peak_tflops": FP64_PEAK_TFLOPS, "fp64_peak_src": "measured DMMA issue rate, tools/fp64_peak"}
    line = {
        "metric": METRIC, "value": value, "unit": "KP-approx/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "step_ms": {"min": float(min(step_ms)), "median": float(np.median(step_ms)), "max": float(max(step_ms)),
                    "all": [round(float(t), 4) for t in step_ms]},
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(n), "parallelism": f"replicas x{world}",
        "result": trace_result(tr) | {"engine": "egkb(arithmetic='fast')",
                                      "note": "fixed-rank config: the fp32 recurrence breaks down past the numerical "
                                              "rank (sigma_i < 1e-6 sigma_1), where the stopping step depends on the "
                                              "last bits of the dot products -- the reference itself stops at k_p = 12 "
                                              "with OpenBLAS's SkylakeX sdot kernel and 11 with the Haswell one; the "
                                              "engine that repeats its roundings bit for bit is under "
                                              "reference_arithmetic; decisions by the nu rule (configs[1], configs[4]) "
                                              "are identical in both engines"},
        "reference_arithmetic": ref_arith_line,
        "roofline": {"kernel": names[dom], "bound": "hbm", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": ncu_traffic(dom), "launches": d_n,
                     "share_of_step": step_share, "peak_src": hbm_src,
                     "timing": "CUDA events around every launch in a replay of the timed steps on the launching "
                               "stream (the same kernels: one persistent eGKB launch per approximation)",
                     "profiled_ms_per_step": prof_ms / args.steps},
        "ra_matvec": ra,
        "sb": sb,
        "sweep": sweep,
        "other_configs": others,
        "sharded_egkb": sharded,
        "e2e": {"value": e2e_value, "unit": "KP-approx/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": float(np.mean(e2e_ms)),
                "step_ms": {"min": float(min(e2e_ms)), "median": float(np.median(e2e_ms)), "max": float(max(e2e_ms))},
                "result_location": "Kronecker factors device-resident (KroneckerSum on the GPU, consumed there "
                                   "by sb_run); sigma and the trace read back to the host",
                "host_factors": {"ms_per_step": float(np.mean(e2e_host_ms)),
                                 "value": world * 1e3 / float(np.mean(e2e_host_ms)),
                                 "d2h_bytes_per_step": int(d2h + host_fac_bytes),
                                 "note": "same call plus op.ax / op.ay: the factors as host fp64 C-ordered "
                                         "n x n arrays (kronop.py:42-43)"}},
        "gpu_launches": int(gpu_launches),
        "clocks": clk,
    }
    # N1 (north_star target): the n=1024 approximation followed by the 200-iteration
    # isotropic SB solve on its factors, end to end on the device
    line["n1"] = {"approx_ms": ms_per_step, "sb_ms": sb_ms, "total_s": (ms_per_step + sb_ms) * 1e-3,
                  "sb_outer_iters": sb_res.outer_iters, "cgls_iters_total": cg,
                  "outer_it_per_s": sb_res.outer_iters / (sb_ms * 1e-3), "cgls_it_per_s": cg / (sb_ms * 1e-3),
                  "final_rc": float(sb_res.rc_history[-1]) if sb_res.rc_history else None,
                  "workload": f"egkb+assemble (k={op.k}) then sb_run isotropic, l_max={sb_res.outer_iters}, "
                              "tau=0, CglsConfig(100, 1e-4), lam=0.1150, beta=0.0066"}
    if split_line is not None:
        line["n1"]["toeplitz_split"] = split_line
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(prob)
        line["cpu_baseline"] = cpu
        line["n1"]["cpu_extrapolated_s"] = cpu["egkb_s"] + cg * cpu["cgls_s_per_it"]
        line["n1"]["cpu_note"] = ("EXTRAPOLATED: the port's measured eGKB time + the GPU run's CGLS iteration "
                                  "count x the port's measured seconds per CGLS iteration (SURVEY §8d)")
    print(json.dumps(line))


def ncu_traffic(cls):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed `ncu --set full` capture (profiles/)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(str(cls))
    except Exception:
        return None


def cpu_baseline(prob):
    from types import SimpleNamespace

    from oracle import lowrank as olr
    from oracle import sb as osb
    from oracle import structured as ost

    n = prob.n
    k32 = psf_f32(prob.psf)
    cfg = SimpleNamespace(reorth=None, seed=0, break_tol=None, keep_basis=False, **egkb_cfg_kwargs())
    t0 = time.perf_counter()
    (u, s, v), tr = olr.egkb(lambda q: ost.ra_matvec(k32, n, q), lambda x: ost.ra_rmatvec(k32, n, x),
                             (n * n, n * n), np.float32, cfg)
    t_egkb = time.perf_counter() - t0
    ax = [s[i].astype(np.float64) * u[:, i].astype(np.float64).reshape((n, n), order="F") for i in range(s.size)]
    ay = [v[:, i].astype(np.float64).reshape((n, n), order="F") for i in range(s.size)]
    op = osb.KronOracle(ax, ay, n, n, n, n)
    aug = osb.AugOracle(op, n, 0.1150, 0.1150)
    rhs = np.concatenate([prob.b, np.zeros(2 * n * (n - 1))])
    t0 = time.perf_counter()
    osb.cgls(aug, rhs, i_max=2, tau=0.0)
    t_cg = (time.perf_counter() - t0) / 2.5   # 1 initial transpose + 2 x (forward + transpose)
    return {"value": 1.0 / t_egkb, "unit": "KP-approx/s", "cores": os.cpu_count(), "kind": "port",
            "sample": "one full eGKB+assemble at n=1024 (oracle restatement, numpy structured R(A)); "
                      f"SB: 2 CGLS iterations of the k={s.size} augmented system",
            "egkb_s": t_egkb, "cgls_s_per_it": t_cg, "cgls_it_per_s": 1.0 / t_cg, "result": trace_result(tr)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sb-outer", type=int, default=200)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2410_00233_b200 import datagen

    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, datagen.make_problem(CONFIG))
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        tdist.init_process_group("nccl")
        dist = tdist
    else:
        torch.cuda.set_device(0)
    prob = datagen.make_problem(CONFIG)
    run_ours(args, prob, rank, world, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
