"""Device Gaussian draws == numpy's default_rng(seed).standard_normal (lowrank.py:199-201, 361-362)."""
import os
import re
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_2410_00233_b200", "csrc", "kb_ziggurat_tables.h")


def _header_tables():
    txt = open(HDR).read()
    out = {}
    for name in ("kKi", "kWi", "kFi"):
        body = re.search(name + r"\[256\] = \{(.*?)\};", txt, re.S).group(1)
        toks = [t.strip() for t in body.replace("\n", " ").split(",") if t.strip()]
        if name == "kKi":
            out[name] = np.array([int(t.rstrip("ULL"), 16) for t in toks], dtype=np.uint64)
        else:
            out[name] = np.array([float.fromhex(t) for t in toks], dtype=np.float64)
    return out


def test_committed_tables_reproduce_numpy():
    """The header's ziggurat tables + the restated algorithm give numpy's draws bit for bit."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_ziggurat as gz

    t = _header_tables()
    _, ki, wi, fi = gz.locate()
    assert np.array_equal(t["kKi"], ki)
    assert np.array_equal(t["kWi"].view(np.uint64), wi.view(np.uint64))
    assert np.array_equal(t["kFi"].view(np.uint64), fi.view(np.uint64))
    gz.verify(t["kKi"], t["kWi"], t["kFi"], seeds=(3, 2024), count=60_000)


def test_pcg64_state_of_default_rng():
    from paper_2410_00233_b200.rng import pcg64_state

    s, inc = pcg64_state(5)
    st = np.random.default_rng(5).bit_generator.state["state"]
    assert (s, inc) == (st["state"], st["inc"])
    with pytest.raises(TypeError):
        pcg64_state(np.random.MT19937(1))


@pytest.mark.gpu
@pytest.mark.parametrize("count", [1, 7, 255, 256, 257, 1000, 65_536 + 13, 1_048_576])
@pytest.mark.parametrize("seed", [0, 1, 12345])
def test_f32_matches_numpy(seed, count):
    from paper_2410_00233_b200.rng import standard_normal

    ref = np.random.default_rng(seed).standard_normal(count).astype(np.float32)
    got = standard_normal(seed, count, np.float32).cpu().numpy()
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("ne", [1, 2, 3])
def test_serial_resolution_path(ne):
    """Fewer speculative entries force the walk's serial re-parse; the stream must not change."""
    from paper_2410_00233_b200 import _lib
    from paper_2410_00233_b200.rng import standard_normal

    lib = _lib.load()
    lib.kb_normal_test_entries(ne)
    try:
        for seed in (2, 99):
            ref = np.random.default_rng(seed).standard_normal(300_001).astype(np.float32)
            got = standard_normal(seed, 300_001, np.float32).cpu().numpy()
            assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))
    finally:
        lib.kb_normal_test_entries(0)


@pytest.mark.gpu
def test_f64_matches_numpy_outside_tail():
    """f64 draws: bit-exact except possibly the last ulp of tail samples (|x| > r)."""
    from paper_2410_00233_b200.rng import standard_normal

    for seed in range(4):
        ref = np.random.default_rng(seed).standard_normal(2_000_000)
        got = standard_normal(seed, 2_000_000, np.float64).cpu().numpy()
        diff = ref != got
        assert np.all(np.abs(ref[diff]) > 3.6541528853610088)
        np.testing.assert_allclose(got[diff], ref[diff], rtol=4e-16, atol=0)


@pytest.mark.gpu
def test_transposed_matrix_layout():
    """cols > 0: the transpose of the row-major draw matrix (RSVD test matrix, lowrank.py:362)."""
    from paper_2410_00233_b200.rng import standard_normal

    ref = np.random.default_rng(8).standard_normal((4099, 30)).astype(np.float32)
    got = standard_normal(8, (4099, 30), np.float32, transpose=True).cpu().numpy()
    assert got.shape == (30, 4099)
    assert np.array_equal(ref.T, got)


@pytest.mark.gpu
def test_seedsequence_and_many_seeds():
    from paper_2410_00233_b200.rng import standard_normal

    ss = np.random.SeedSequence(271828)
    ref = np.random.default_rng(ss).standard_normal(50_000).astype(np.float32)
    got = standard_normal(np.random.PCG64(np.random.SeedSequence(271828)), 50_000, np.float32).cpu().numpy()
    assert np.array_equal(ref, got)
    mism = 0
    for seed in range(40):
        ref = np.random.default_rng(seed).standard_normal(262_144).astype(np.float32)
        got = standard_normal(seed, 262_144, np.float32).cpu().numpy()
        mism += int(np.sum(ref.view(np.uint32) != got.view(np.uint32)))
    assert mism == 0
