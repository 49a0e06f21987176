"""Multi-GPU partitioning: Kronecker-term sharding of the SB solve.

One process per GPU.  A :class:`ShardedKroneckerSum` holds this rank's
contiguous slice of the k Kronecker terms; every product of the operator is a
rank-local partial sum (two DMMA GEMMs over k/G terms) followed by ONE
sum-allreduce of the n^2 fp64 result, issued from inside the CGLS loop of
``kb_cgls_run`` / ``kb_sb_run`` through the ``kb_allreduce_fn`` hook of the C
ABI, stream-ordered on the current stream (NCCL over NVLink on a B200 box).
All vector work stays replicated, so every rank holds the same iterate and
makes the same stop decisions.

With an NCCL process group the hook is the library's C function
``kb_nccl_allreduce_f64`` on torch's communicator (no Python callback inside the
solve); other backends (gloo) use a Python callback.

The eGKB side is row-sharded (:func:`sharded_egkb`): each rank
owns a contiguous block of image rows of every Krylov vector, K is replicated,
and the per-half-step cross-shard sums (diagonal sums, reorthogonalisation
coefficients, norms) are exact integer-limb partials combined by one int64
sum-allreduce each -- so the recurrence is bit-identical for any shard count
(``kb_egkb_shard.cu``).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib
from .kronop import KroneckerSum


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of ``total`` items for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class _BufferRegistry:
    """Maps raw device pointers handed to the allreduce hook back to torch views."""

    def __init__(self):
        self._tensors: list[torch.Tensor] = []

    def add(self, t: torch.Tensor):
        self._tensors.append(t)

    def remove(self, t: torch.Tensor):
        self._tensors = [x for x in self._tensors if x is not t]

    def view(self, ptr: int, count: int) -> torch.Tensor:
        from . import device as D

        cands = list(self._tensors)
        ws = D.WORKSPACE._buf.get(D.device().index or 0)
        if ws is not None:
            cands.append(ws)
        for t in cands:
            base = t.data_ptr()
            nbytes = t.numel() * t.element_size()
            if base <= ptr and ptr + 8 * count <= base + nbytes:
                off = ptr - base
                return t.view(torch.uint8).reshape(-1)[off:off + 8 * count].view(torch.float64)
        raise RuntimeError("allreduce hook: buffer is not a registered device tensor")


REGISTRY = _BufferRegistry()


class ShardedKroneckerSum:
    """This rank's share of a KroneckerSum; products are summed across ``group``."""

    def __init__(self, full: KroneckerSum, group=None):
        import torch.distributed as dist

        self.full = full
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        lo, hi = shard_range(full.k, self.world, self.rank)
        if hi <= lo:
            raise ValueError(f"rank {self.rank} owns no Kronecker terms (k={full.k}, world={self.world})")
        self.terms = (lo, hi)
        self.scheme = full.scheme
        self.f_dev = full.f_dev[lo:hi]
        self.g_dev = full.g_dev[lo:hi]
        self._hook = _lib.ALLREDUCE_FN(self._allreduce)
        self._ctx = None
        self._nccl_comm = None
        if dist.is_initialized() and dist.get_backend(group) == "nccl":
            # the C hook over NCCL on torch's own communicator: no Python inside the solve
            pg = group if group is not None else dist.distributed_c10d._get_default_group()
            backend = pg._get_backend(torch.device("cuda"))
            t = torch.zeros(1, dtype=torch.float64, device="cuda")
            dist.all_reduce(t, group=group)   # the communicator exists after a first collective
            comm = backend._comm_ptr()
            lib = _lib.load()
            if comm and lib.kb_nccl_available():
                self._nccl_comm = comm
                self._hook = C.cast(lib.kb_nccl_allreduce_f64, _lib.ALLREDUCE_FN)
                self._ctx = C.c_void_p(comm)

    def _allreduce(self, ctx, buf, count, stream):
        import torch.distributed as dist

        if self.world == 1:
            return
        view = REGISTRY.view(C.cast(buf, C.c_void_p).value, int(count))
        dist.all_reduce(view, op=dist.ReduceOp.SUM, group=self.group)

    @property
    def k(self) -> int:
        return self.terms[1] - self.terms[0]

    @property
    def shape(self):
        return self.full.shape

    def forward_struct(self) -> _lib.KbForward:
        s = self.scheme
        fw = _lib.KbForward()
        fw.kind = _lib.KB_FWD_KRON
        fw.m, fw.n = self.shape
        fw.a, fw.lda = None, 0
        fw.kron = _lib.KbKron(s.m1, s.m2, s.n1, s.n2, self.k, self.f_dev.data_ptr(), self.g_dev.data_ptr())
        if hasattr(self.full, "kron_struct"):   # the full sum's G band bounds every term subset's
            full = self.full.kron_struct()
            fw.kron.band = full.band
            if full.fband:   # a Toeplitz-split sum: its F band bounds every subset of the banded terms
                nd = max(0, min(full.ndense - self.terms[0], self.k))   # dense terms lead the full sum
                fw.kron.ndense = nd
                fw.kron.fband = full.fband
                if nd > 0 and full.ft:
                    fw.kron.ft = full.ft + 8 * self.terms[0] * s.n1 * s.m1
            elif full.ft:   # this rank's F^T blocks: the transposed reduced stage as one GEMM too
                fw.kron.ft = full.ft + 8 * self.terms[0] * s.n1 * s.m1
        fw.allreduce = self._hook
        fw.allreduce_ctx = self._ctx
        return fw

    def apply(self, x, counter=None):
        from .kronop import _forward_apply

        return _forward_apply(self.forward_struct(), x, 0, self.shape)

    def apply_t(self, y, counter=None):
        from .kronop import _forward_apply

        return _forward_apply(self.forward_struct(), y, 1, self.shape)


# ----------------------------------------------------------------- row-sharded eGKB
_SHARD_CACHE: dict = {}

class _Shards:
    """Which 8-row blocks of the n x n image each shard owns, and how partial limb
    buffers are combined: in place by an int64 sum-allreduce over ``group`` (one
    shard per rank), or -- ``simulate=G`` on one device -- by running all G shards'
    kernels into the same buffer (limb additions are exact, so this IS the
    allreduce's result)."""

    def __init__(self, n, group=None, simulate=None):
        import torch.distributed as dist

        nblk = -(-n // 8)
        if simulate:
            self.world, self.mine, self.group = int(simulate), list(range(int(simulate))), None
        else:
            self.world = dist.get_world_size(group) if dist.is_initialized() else 1
            rank = dist.get_rank(group) if dist.is_initialized() else 0
            self.mine, self.group = [rank], group
        self.ranges = []
        for g in range(self.world):
            lo, hi = shard_range(nblk, self.world, g)
            self.ranges.append((min(8 * lo, n), min(8 * hi, n)))
        self.simulated = bool(simulate)

    def own(self):
        return [self.ranges[g] for g in self.mine]

    def allreduce(self, t):
        import torch.distributed as dist

        if not self.simulated and self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def uniform(self):
        """Every shard holds the same number of rows (the gather path applies)."""
        return len({a1 - a0 for a0, a1 in self.ranges}) == 1

    def allgather(self, t):
        """[G, *t.shape]: every rank's t in rank order (NCCL: one all_gather_into_tensor)."""
        import torch.distributed as dist

        if dist.get_backend(self.group) == "nccl":
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.stack(parts)


class CudaShardKernels:
    """The per-shard steps of the sharded recurrence: ``kb_shard_*`` (kb_egkb_shard.cu) on
    the current CUDA stream.  Every method takes torch tensors; integer limb buffers are
    accumulated into (the caller zeroes them)."""

    def __init__(self):
        from . import device as D

        self.lib = _lib.load()
        self.device = D.device()
        self._st = D.stream_ptr

    def _check(self, rc, what):
        _lib.check(rc, what)

    def sqnorm(self, x, n, a0, a1, nl):
        self._check(self.lib.kb_shard_sqnorm(x.data_ptr(), n, a0, a1, nl.data_ptr(), self._st()), "shard sqnorm")

    def z(self, Mt, wl, z):
        """z = Mt w (Mt: cols x rows; one row dot per output)."""
        cols, rows = Mt.shape
        self._check(self.lib.kb_shard_z(Mt.data_ptr(), rows, cols, wl.data_ptr(), z.data_ptr(), self._st()),
                    "shard z")

    def bcast_dots(self, z, n, c, length, beta, prev, B, m, a0, a1, v, dl):
        self._check(self.lib.kb_shard_bcast_dots(z.data_ptr(), n, c, length, beta.data_ptr(),
                                                 prev.data_ptr() if prev is not None else None, B.data_ptr(),
                                                 B.shape[1], m, a0, a1, v.data_ptr(), dl.data_ptr(), self._st()),
                    "shard dots")

    def update(self, v, B, m, dl, n, a0, a1, nl, scal):
        self._check(self.lib.kb_shard_update(v.data_ptr(), B.data_ptr(), B.shape[1], m, dl.data_ptr(), n, a0, a1,
                                             nl.data_ptr(), scal.data_ptr(), self._st()), "shard update")

    def normalize(self, src, nl, out, n, c, length, a0, a1, wl, scal):
        self._check(self.lib.kb_shard_normalize(src.data_ptr(), nl.data_ptr(), out.data_ptr(), n, c, length, a0, a1,
                                                wl.data_ptr(), scal.data_ptr(), self._st()), "shard normalize")

    def lift(self, B, rows, W, out, off, ln, out_off=None):
        """out[:, o:o+ln] = W[:rows].T @ B[:rows, off:off+ln] with o = off, or out_off when given
        (kb_ts_lift on a row slice; out's own row stride)."""
        if ln == 0:
            return
        N = B.shape[1]
        o = off if out_off is None else out_off
        self._check(self.lib.kb_ts_lift(_lib.KB_F32, B.data_ptr() + 4 * off, N, rows, W.data_ptr(), W.shape[1],
                                        out.data_ptr() + 4 * o, out.shape[1], ln, self._st()), "shard lift")


def sharded_egkb(b_mat, config, y0=None, *, group=None, simulate=None, kernels=None):
    """eGKB (lowrank.py:159-329) with the Krylov vectors row-sharded across the ranks of
    ``group`` (one GPU each), or across ``simulate`` virtual shards on one device.

    Same trace semantics, breakdown tests and nu rule as :func:`egkb`; the arithmetic is
    the sharded engine's own (per-chunk fp64 partials, exact integer combination), so the
    result does not depend on the number of shards.  fp32, zero-BC ``RearrangedBlur``.
    Returns ``(TruncatedSvd, EgkbTrace)`` with the singular vectors on every rank.
    ``kernels`` replaces the CUDA shard steps (tests drive this host loop and its
    allreduce protocol with a host implementation over gloo).
    """
    import numpy as np

    from . import rng
    from .blurmodel import BC_ZERO, RearrangedBlur
    from .exceptions import NumericalError, ValidationError
    from .linalg import TruncatedSvd
    from .lowrank import EgkbTrace, eps_for

    if not isinstance(b_mat, RearrangedBlur) or b_mat.bc != BC_ZERO or b_mat.dtype != np.float32:
        raise ValidationError("sharded_egkb needs a float32 zero-BC RearrangedBlur")
    kern = kernels if kernels is not None else CudaShardKernels()
    dev = kern.device
    n = b_mat.n
    N = n * n
    kh, kw = b_mat.psf.shape
    cu, cv = kh // 2, kw // 2
    if kernels is None:
        K, Kt = b_mat._device_kernels()
    else:
        k32 = torch.from_numpy((b_mat.psf.kernel).astype(np.float32))
        K, Kt = k32.to(dev), k32.t().contiguous().to(dev)
    sh = _Shards(n, group, simulate)
    tol = config.break_tol if config.break_tol is not None else float(np.sqrt(eps_for(np.float32)))
    cap = max(config.k_max, config.k_min) + config.p + 3
    # persistent state per (device, shape, shards, kernel): the buffers, and -- from the second
    # call on -- one CUDA graph per half step (the per-shard launches, the limb zeroing and,
    # across ranks, the NCCL allreduces), replayed instead of re-launched from Python
    ckey = None
    if kernels is None:
        ckey = (dev.index, n, kh, kw, cap, sh.world, tuple(sh.mine), K.data_ptr(), Kt.data_ptr(), id(group))
    st = _SHARD_CACHE.get(ckey) if ckey is not None else None
    if st is None:
        st = {"S": torch.zeros((cap, N), dtype=torch.float32, device=dev),
              "Q": torch.zeros((cap, N), dtype=torch.float32, device=dev),
              "v": torch.zeros((N,), dtype=torch.float32, device=dev),
              "y0": torch.zeros((N,), dtype=torch.float32, device=dev),
              "z": torch.zeros(kh + kw + 8, dtype=torch.float64, device=dev),
              # all limb accumulators in one buffer (one fill per half step): w | dots | norm
              "limbs": torch.zeros(3 * (max(kh, kw) + 8) + 3 * (cap + 3) + 3, dtype=torch.int64, device=dev),
              # per half step (t or alpha, |y|), written by the kernels; the next half step's
              # beta is the previous row's first entry
              "hist": torch.zeros((2 * cap + 2, 2), dtype=torch.float64, device=dev),
              "graphs": {}, "calls": 0}
        if ckey is not None:
            if len(_SHARD_CACHE) >= 4:
                _SHARD_CACHE.pop(next(iter(_SHARD_CACHE)))
            _SHARD_CACHE[ckey] = st
    st["calls"] += 1
    use_graphs = ckey is not None and st["calls"] >= 2 and not os.environ.get("KB_SHARD_NO_GRAPH")
    S, Q, v, z, limbs = st["S"], st["Q"], st["v"], st["z"], st["limbs"]
    lw = 3 * (max(kh, kw) + 8)
    wl, dl, nl = limbs[:lw], limbs[lw:lw + 3 * (cap + 3)], limbs[lw + 3 * (cap + 3):]
    hist, graphs = st["hist"], st["graphs"]
    if y0 is None:
        y0src = rng.standard_normal(config.seed, N, np.float32)
    elif isinstance(y0, torch.Tensor):
        y0src = y0.to(device=dev, dtype=torch.float32).reshape(-1)
    else:
        y0src = torch.from_numpy(np.ascontiguousarray(y0, dtype=np.float32)).to(dev).reshape(-1)
    if tuple(y0src.shape) != (N,):
        raise ValidationError(f"y0 must have length {N}, got shape {tuple(y0src.shape)}")
    y0d = st["y0"]
    y0d.copy_(y0src)

    def run(gkey, fn):
        if not use_graphs:
            fn()
            return
        g = graphs.get(gkey)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            graphs[gkey] = g
        g.replay()

    def normalize(src, out, c_next, len_next, scal):
        """t = |src| (allreduced limbs in nl) -> out = fl(src / t), next product's diagonal limbs."""
        for a0, a1 in sh.own():
            kern.normalize(src, nl, out, n, c_next, len_next, a0, a1, wl, scal)
        sh.allreduce(wl)

    def half(Mt, c_b, len_b, prev, B, m, out, c_next, len_next, slot):
        """One half step (R q or R^T s): z from the all-reduced diagonal limbs; y, v = y - beta prev
        and the limbs of B^T v, |v|^2, |y|^2; v1 = v - B h and the limbs of |v1|^2; out = v1 / t
        and the next product's diagonal limbs.  (t or alpha, |y|) land in hist[slot]; beta is the
        previous half step's t or alpha (hist[slot - 1, 0])."""
        kern.z(Mt, wl, z)
        limbs.zero_()   # w was consumed by z; the dot and norm limbs were consumed last half step
        beta = hist[slot - 1, :1]
        for a0, a1 in sh.own():
            kern.bcast_dots(z, n, c_b, len_b, beta, prev, B, m, a0, a1, v, dl)
        sh.allreduce(dl[: 3 * (m + 2)])
        for a0, a1 in sh.own():
            kern.update(v, B, m, dl, n, a0, a1, nl, hist[slot])
        sh.allreduce(nl)
        normalize(v, out, c_next, len_next, hist[slot])

    def init():
        # s1 = y0 / |y0|, diagonal limbs for R^T s1 (lowrank.py:207-210)
        limbs.zero_()
        for a0, a1 in sh.own():
            kern.sqnorm(y0d, n, a0, a1, nl)
        sh.allreduce(nl)
        normalize(y0d, S[0], cv, kw, hist[0])
        # q1 = R^T s1 / alpha1 (lowrank.py:211-215): no previous vector, no projection
        half(K, cu, kh, None, Q, 0, Q[0], cu, kh, 1)

    run(("init",), init)
    h = hist[:2].cpu().numpy()
    t1, a1 = float(h[0, 0]), float(h[1, 0])
    if t1 == 0.0:
        raise ValidationError("starting vector must be nonzero")
    if a1 == 0.0:
        raise NumericalError("operator annihilates the starting vector")
    trace = EgkbTrace()
    trace.alphas, trace.ts, trace.zetas, trace.nus = [a1], [t1], [a1 * t1], [1e308]
    fired, reason, done = None, "", 1
    broke = t_break = False
    while done < ((fired + config.p + 1) if fired is not None else (config.k_max + 1)):
        if done + 1 > cap:
            raise NumericalError("eGKB basis capacity exhausted")
        slot = 2 * done
        # s step: u = R q_j, s_raw = u - alpha s_j, projected against S (lowrank.py:238-247)
        ms = done if config.reorth != "one-sided" else 0
        run(("s", done, ms), lambda: half(Kt, cv, kw, S[done - 1], S, ms, S[done], cv, kw, slot))
        # q step: R^T s_{j+1} - t q_j, projected against Q (lowrank.py:250-260)
        run(("q", done), lambda: half(K, cu, kh, Q[done - 1], Q, done, Q[done], cu, kh, slot + 1))
        h = hist[slot:slot + 2].cpu().numpy()
        t_new, u_norm, a_new, pre = float(h[0, 0]), float(h[0, 1]), float(h[1, 0]), float(h[1, 1])
        if t_new <= tol * u_norm:
            broke = t_break = True
            break
        if a_new <= tol * pre:
            broke = True
            trace.ts.append(t_new)
            break
        trace.ts.append(t_new)
        trace.alphas.append(a_new)
        zeta = a_new * t_new
        nu = float(np.sqrt(zeta * trace.zetas[-1]))
        trace.zetas.append(zeta)
        trace.nus.append(nu)
        done += 1
        if fired is None:
            if nu > trace.nus[-2]:
                fired, reason = max(done - 1, config.k_min), "nu_rose"
            elif nu < config.tau:
                fired, reason = max(done, config.k_min), "nu_below_tol"
    if broke:
        k_p, rows = done, (done if t_break else done + 1)
    else:
        k_p, rows = done - 1, done
    if fired is not None:
        chosen = min(fired, k_p)
    elif broke:
        chosen, reason = k_p, "breakdown"
    else:
        chosen, reason = min(config.k_max, k_p), "hit_kmax"
    if chosen < 1 or k_p < 1:
        raise NumericalError("bidiagonalization broke down before producing any factors")
    c_mat = np.zeros((rows, k_p))
    for i in range(k_p):
        c_mat[i, i] = np.float32(trace.alphas[i])
        if i + 1 < rows:
            c_mat[i + 1, i] = np.float32(trace.ts[i + 1])
    uc, sc, vct = np.linalg.svd(c_mat, full_matrices=False)
    sigma = sc[:chosen].astype(np.float32).astype(np.float64)
    # lift on the own rows (lowrank.py:317-318), then the rows of the other ranks
    wu = torch.from_numpy(np.ascontiguousarray(uc[:, :chosen], dtype=np.float32)).to(dev)
    wv = torch.from_numpy(np.ascontiguousarray(vct.T[:, :chosen], dtype=np.float32)).to(dev)
    if sh.simulated or sh.world == 1:   # this process lifts every row
        out_u = torch.empty((chosen, N), dtype=torch.float32, device=dev)
        out_v = torch.empty((chosen, N), dtype=torch.float32, device=dev)
        for a0, a1 in sh.own():
            kern.lift(S, rows, wu, out_u, a0 * n, (a1 - a0) * n)
            kern.lift(Q, k_p, wv, out_v, a0 * n, (a1 - a0) * n)
    elif sh.uniform():                  # own rows lifted into a slab, the slabs all-gathered
        (a0, a1), = sh.own()
        ln = (a1 - a0) * n
        slab = torch.empty((2, chosen, ln), dtype=torch.float32, device=dev)
        kern.lift(S, rows, wu, slab[0], a0 * n, ln, out_off=0)
        kern.lift(Q, k_p, wv, slab[1], a0 * n, ln, out_off=0)
        g = sh.allgather(slab)            # [G, 2, chosen, ln]: rank r holds rows [r ln/n, (r+1) ln/n)
        out_u = g[:, 0].permute(1, 0, 2).reshape(chosen, N)
        out_v = g[:, 1].permute(1, 0, 2).reshape(chosen, N)
    else:                               # uneven shards: zeros outside the own rows, summed
        out_u = torch.zeros((chosen, N), dtype=torch.float32, device=dev)
        out_v = torch.zeros((chosen, N), dtype=torch.float32, device=dev)
        for a0, a1 in sh.own():
            kern.lift(S, rows, wu, out_u, a0 * n, (a1 - a0) * n)
            kern.lift(Q, k_p, wv, out_v, a0 * n, (a1 - a0) * n)
        sh.allreduce(out_u)
        sh.allreduce(out_v)
    trace.chosen_k, trace.k_p, trace.stop_reason, trace.breakdown = chosen, k_p, reason, broke
    return TruncatedSvd.from_device(out_u, sigma.astype(np.float32), out_v), trace
