"""World-size-2 gloo tests (CPU) of the multi-GPU partition and reduction
protocol used by paper_2410_00233_b200.parallel: Kronecker-term
sharding with one sum-allreduce per operator product.  The per-rank compute
here is the CPU oracle (test infrastructure); on a B200 box the same
partition drives the DMMA kernels and the allreduce hook runs NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sb as osb
        from paper_2410_00233_b200.parallel import shard_range

        rng = np.random.default_rng(7)
        n, k = 12, 5
        ax = [rng.standard_normal((n, n)) for _ in range(k)]
        ay = [rng.standard_normal((n, n)) for _ in range(k)]
        full = osb.KronOracle(ax, ay, n, n, n, n)
        lo, hi = shard_range(k, world, rank)
        local = osb.KronOracle(ax[lo:hi], ay[lo:hi], n, n, n, n)

        class Sharded:
            shape = full.shape

            def _sum(self, v):
                t = torch.from_numpy(np.ascontiguousarray(v))
                dist.all_reduce(t)
                return t.numpy()

            def apply(self, x):
                return self._sum(local.apply(x))

            def apply_t(self, y):
                return self._sum(local.apply_t(y))

        x = rng.standard_normal(n * n)
        err_apply = np.abs(Sharded().apply(x) - full.apply(x)).max()
        err_t = np.abs(Sharded().apply_t(x) - full.apply_t(x)).max()
        b = rng.standard_normal(n * n)
        ref = osb.sb_run(full, b, 0.115, 0.0066, variant="isotropic", tau=0.0, l_max=3, i_max=15, tau_cgls=0.0)
        got = osb.sb_run(Sharded(), b, 0.115, 0.0066, variant="isotropic", tau=0.0, l_max=3, i_max=15,
                         tau_cgls=0.0)
        gap = np.linalg.norm(got.x - ref.x) / np.linalg.norm(ref.x)
        q.put((rank, (lo, hi), float(err_apply), float(err_t), float(gap), got.cgls_iters == ref.cgls_iters))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_term_sharded_sb_protocol_world2():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    assert res[0][1] == (0, 3) and res[1][1] == (3, 5)
    for _, _, ea, et, gap, same in res:
        assert ea < 1e-12 and et < 1e-12
        assert gap < 1e-12
        assert same


def test_shard_range_partitions():
    from paper_2410_00233_b200.parallel import shard_range

    for total in (1, 5, 13, 30):
        for world in (1, 2, 4, 8):
            if world > total:
                continue
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1
