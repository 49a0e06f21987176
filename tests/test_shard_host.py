"""The row-sharded eGKB host loop (paper_2410_00233_b200.parallel.sharded_egkb,
SURVEY §8e) on CPU: partition invariance with simulated shards and a real
world-size-2 gloo run, the per-shard steps supplied by tests/shard_host_kernels.py
(the device steps are covered by tests/test_gpu_shard.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_SIDE = 48


def _problem(side=N_SIDE):
    from paper_2410_00233_b200 import datagen

    psf = datagen.mixture_psf(side, seed=5)
    y0 = np.random.default_rng(0).standard_normal(side * side).astype(np.float32)
    return psf, y0


def _run(group=None, simulate=None, side=N_SIDE):
    import paper_2410_00233_b200 as kb
    from paper_2410_00233_b200.parallel import sharded_egkb
    from shard_host_kernels import HostShardKernels

    psf, y0 = _problem(side)
    svd, tr = sharded_egkb(kb.RearrangedBlur(psf, side), kb.EgkbConfig(k_max=12), y0=y0, group=group,
                           simulate=simulate, kernels=HostShardKernels())
    return tr, np.asarray(svd.sigma), svd._u_dev.numpy().copy(), svd._v_dev.numpy().copy()


def test_partition_invariance_simulated():
    ref = _run(simulate=1)
    assert ref[0].k_p >= 3
    for g in (2, 3, 6):
        tr, s, u, v = _run(simulate=g)
        assert (tr.alphas, tr.ts, tr.nus) == (ref[0].alphas, ref[0].ts, ref[0].nus), g
        assert (tr.chosen_k, tr.k_p, tr.stop_reason) == (ref[0].chosen_k, ref[0].k_p, ref[0].stop_reason)
        assert np.array_equal(s, ref[1])
        assert np.allclose(u, ref[2], atol=1e-6) and np.allclose(v, ref[3], atol=1e-6)


def test_shard_rows_cover_the_image():
    from paper_2410_00233_b200.parallel import _Shards

    for n in (8, 48, 100, 1024):
        for g in (1, 2, 3, 8):
            r = _Shards(n, simulate=g).ranges
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert all(a0 % 8 == 0 for a0, _ in r)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, side, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr, s, u, v = _run(side=side)
        q.put((rank, tr.alphas, tr.ts, tr.k_p, tr.chosen_k, s.tolist(), u, v))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("side", [48, 40])   # 6 row blocks (even shards: gathered slabs), 5 (uneven: summed)
def test_world2_gloo_matches_single_shard(side):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, side, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get() for _ in range(2)), key=lambda r: r[0])   # drained before join (large payloads)
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    ref = _run(simulate=1, side=side)
    for rank, alphas, ts, k_p, chosen, s, u, v in res:
        assert alphas == ref[0].alphas and ts == ref[0].ts, rank
        assert (k_p, chosen) == (ref[0].k_p, ref[0].chosen_k)
        assert s == ref[1].tolist()
        # every rank holds every row of the singular vectors
        np.testing.assert_allclose(u, ref[2], atol=1e-6)
        np.testing.assert_allclose(v, ref[3], atol=1e-6)


def test_limb_decode_matches_the_library():
    """kb_shard_limbs_value (the device formula, host-callable) decodes like the host helper,
    and to_limbs / from_limbs round-trip values to 2^-79."""
    import ctypes

    from paper_2410_00233_b200 import _lib
    from shard_host_kernels import from_limbs, to_limbs

    lib = _lib.load()
    rng = np.random.default_rng(1)
    for x in np.concatenate([rng.standard_normal(50) * 10.0 ** rng.uniform(-20, 10, 50), [0.0, 1.0, -3.5]]):
        limbs = to_limbs(x)
        assert abs(from_limbs(*limbs) - x) <= 2.0 ** -78 + 1e-15 * abs(x)
        arr = (ctypes.c_longlong * 3)(*[int(v) for v in limbs])
        assert lib.kb_shard_limbs_value(arr) == from_limbs(*limbs)
