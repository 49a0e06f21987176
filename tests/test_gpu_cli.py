"""CLI on the GPU path (cli.py:318-527) vs the reference CLI's own outputs
(tests/golden/cli, written by running the reference CLI on the same inputs)."""

import csv
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
CLI = os.path.join(GOLDEN, "cli")


@pytest.fixture(scope="module")
def work(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")
    for f in ("psf.mtx", "observed.pgm", "truth.pgm", "matrix.mtx"):
        shutil.copy(os.path.join(CLI, f), d / f)
    shutil.copytree(os.path.join(CLI, "approx_double"), d / "ref_approx_double")
    return d


def _run(work, argv):
    from paper_2410_00233_b200 import cli

    cwd = os.getcwd()
    os.chdir(work)
    try:
        return cli.main(argv)
    finally:
        os.chdir(cwd)


def _json(*p):
    with open(os.path.join(*p)) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name,argv", [
    ("approx_single", ["approx", "--psf", "psf.mtx", "--side", "16", "--prec", "single", "--k-max", "10"]),
    ("approx_double", ["approx", "--psf", "psf.mtx", "--side", "16", "--k-max", "8", "--k-min", "8",
                       "--tau-egkb", "1e300"]),
    ("approx_rsvd", ["approx", "--matrix", "matrix.mtx", "--engine", "rsvd", "--k", "3", "--p", "1", "--q", "2"]),
])
def test_approx_matches_reference_cli(work, name, argv):
    from paper_2410_00233_b200 import io as kio

    assert _run(work, argv + ["--out-dir", name]) == 0
    ref, got = os.path.join(CLI, name), os.path.join(work, name)
    rs, gs = _json(ref, "summary.json"), _json(got, "summary.json")
    assert (gs["k"], gs["k_p"], gs["engine"], gs["precision"], gs["scheme"]) == \
        (rs["k"], rs["k_p"], rs["engine"], rs["precision"], rs["scheme"])
    for key, val in rs["config"].items():
        assert gs["config"][key] == val, key
    single = "single" in name
    sig_r = kio.read_mtx(os.path.join(ref, "svd_sigma.mtx"))[:, 0]
    sig_g = kio.read_mtx(os.path.join(got, "svd_sigma.mtx"))[:, 0]
    np.testing.assert_allclose(sig_g, sig_r, rtol=1e-4 if single else 1e-10)
    for key in ("rel_err_rearranged", "rel_err_operator"):
        if single:
            assert gs[key] < 1e-5 and rs[key] < 1e-5           # both at the fp32 floor
        else:
            assert gs[key] == pytest.approx(rs[key], rel=1e-6, abs=1e-13)
    if os.path.exists(os.path.join(ref, "trace.json")):
        rt, gt = _json(ref, "trace.json"), _json(got, "trace.json")
        assert (gt["chosen_k"], gt["k_p"], gt["stop_reason"], gt["breakdown"]) == \
            (rt["chosen_k"], rt["k_p"], rt["stop_reason"], rt["breakdown"])
        np.testing.assert_allclose(gt["alphas"], rt["alphas"], rtol=1e-4 if single else 1e-10)
    # the saved operators agree term by term (kron(ax_i, ay_i) is sign-invariant)
    op_r, meta_r = kio.load_kron_dir(os.path.join(ref, "operator"))
    op_g, meta_g = kio.load_kron_dir(os.path.join(got, "operator"))
    assert {k: meta_g[k] for k in meta_r} == meta_r
    tol = 1e-4 if single else 1e-9
    assert np.linalg.norm(op_g.materialize() - op_r.materialize()) <= tol * np.linalg.norm(op_r.materialize())


def test_kron_dir_written_byte_identical(work, tmp_path):
    from paper_2410_00233_b200 import io as kio

    src = os.path.join(GOLDEN, "io", "kron")
    op, meta = kio.load_kron_dir(src)
    extra = {k: v for k, v in meta.items() if k not in ("k", "scheme")}
    kio.save_kron_dir(op, tmp_path / "kron", extra_meta=extra)
    for f in sorted(os.listdir(src)):
        with open(os.path.join(src, f), "rb") as a, open(tmp_path / "kron" / f, "rb") as b:
            assert a.read() == b.read(), f


def test_deblur_matches_reference_cli(work):
    from paper_2410_00233_b200 import io as kio

    argv = ["deblur", "--operator-dir", "ref_approx_double/operator", "--observed", "observed.pgm", "--truth",
            "truth.pgm", "--lam", "0.1", "--gamma", "2.0", "--l-max", "5", "--tau-sb", "0", "--i-max", "20",
            "--tau-cgls", "0", "--out-dir", "deblur"]     # SURVEY §8c short protocol: the strict bar applies
    assert _run(work, argv) == 0
    rm, gm = _json(CLI, "deblur", "metrics.json"), _json(work, "deblur", "metrics.json")
    for key in ("outer_iters", "stop", "cgls_iters", "iota_total", "variant", "flops"):
        assert gm[key] == rm[key], key
    for key in ("lam", "beta", "gamma"):
        assert gm[key] == pytest.approx(rm[key], rel=1e-15)
    np.testing.assert_allclose(gm["re"], rm["re"], rtol=1e-8)
    np.testing.assert_allclose(gm["rc_sb"], rm["rc_sb"], rtol=1e-6)
    assert gm["snr_db"] == pytest.approx(rm["snr_db"], rel=1e-10)
    a = kio.read_pgm(os.path.join(CLI, "deblur", "restored.pgm"))
    b = kio.read_pgm(os.path.join(work, "deblur", "restored.pgm"))
    assert np.max(np.abs(a - b)) <= 1.0 / 65535 + 1e-15                  # at most one 16-bit LSB


def test_sweep_matches_reference_cli(work):
    argv = ["sweep", "--operator-dir", "ref_approx_double/operator", "--observed", "observed.pgm", "--truth",
            "truth.pgm", "--count", "4", "--lam-min", "0.02", "--lam-max", "0.5", "--l-max", "3", "--tau-sb", "0",
            "--i-max", "20", "--tau-cgls", "0", "--out-dir", "sweep"]
    assert _run(work, argv) == 0

    def rows(p):
        with open(p, newline="") as fh:
            return list(csv.DictReader(fh))

    ref, got = rows(os.path.join(CLI, "sweep", "sweep.csv")), rows(os.path.join(work, "sweep", "sweep.csv"))
    assert len(ref) == len(got) == 4
    for r, g in zip(ref, got):
        assert (g["outer_iters"], g["iota_total"]) == (r["outer_iters"], r["iota_total"])
        for key in ("lam", "beta"):
            assert float(g[key]) == pytest.approx(float(r[key]), rel=1e-15)
        assert float(g["re"]) == pytest.approx(float(r["re"]), rel=1e-8)


def test_exit_codes(work):
    assert _run(work, ["approx", "--psf", "psf.mtx", "--side", "0", "--out-dir", "bad"]) == 2
    assert _run(work, ["approx", "--psf", "psf.mtx", "--side", "16", "--engine", "tsvd", "--k", "3",
                       "--out-dir", "tsvd"]) == 0
    assert _run(work, ["approx", "--matrix", "matrix.mtx", "--sparse", "--prec", "single", "--k-max", "6",
                       "--out-dir", "sparse"]) == 0
