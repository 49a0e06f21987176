"""Multi-GPU partitioning: Kronecker-term sharding of the SB solve.

One process per GPU.  A :class:`ShardedKroneckerSum` holds this rank's
contiguous slice of the k Kronecker terms; every product of the operator is a
rank-local partial sum (two DMMA GEMMs over k/G terms) followed by ONE
sum-allreduce of the n^2 fp64 result, issued from inside the CGLS loop of
``kb_cgls_run`` / ``kb_sb_run`` through the ``kb_allreduce_fn`` hook of the C
ABI, stream-ordered on the current stream (NCCL over NVLink on a B200 box).
All vector work stays replicated, so every rank holds the same iterate and
makes the same stop decisions.

The eGKB side runs as independent replicas in this round.
"""

from __future__ import annotations

import ctypes as C

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
            fw.kron.band = self.full.kron_struct().band
        fw.allreduce = self._hook
        fw.allreduce_ctx = None
        return fw

    def apply(self, x, counter=None):
        from .kronop import _forward_apply

        return _forward_apply(self.forward_struct(), x, 0, self.shape)

    def apply_t(self, y, counter=None):
        from .kronop import _forward_apply

        return _forward_apply(self.forward_struct(), y, 1, self.shape)
