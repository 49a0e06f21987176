"""On-disk formats (io.py:23-152) vs files written by the reference."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

IOD = os.path.join(GOLDEN, "io")


def _bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


@pytest.fixture(scope="module")
def exp():
    with np.load(os.path.join(IOD, "expected.npz")) as f:
        return {k: f[k] for k in f.files}


def test_read_mtx_reference_files(exp):
    from paper_2410_00233_b200 import io as kio

    a = kio.read_mtx(os.path.join(IOD, "m64.mtx"))
    assert a.dtype == np.float64 and np.array_equal(a, exp["m64"])
    b = kio.read_mtx(os.path.join(IOD, "m32.mtx"))
    assert b.dtype == np.float32 and np.array_equal(b, exp["m32"])
    v = kio.read_mtx(os.path.join(IOD, "vec.mtx"))
    assert v.shape == (6, 1) and np.array_equal(v[:, 0], exp["vec"])


def test_write_mtx_byte_identical(exp, tmp_path):
    from paper_2410_00233_b200 import io as kio

    for name in ("m64", "m32", "vec"):
        out = tmp_path / f"{name}.mtx"
        kio.write_mtx(out, exp[name])
        assert _bytes(out) == _bytes(os.path.join(IOD, f"{name}.mtx")), name


def test_pgm_roundtrip_and_bytes(exp, tmp_path):
    from paper_2410_00233_b200 import io as kio

    for depth in (8, 16):
        ref = os.path.join(IOD, f"img{depth}.pgm")
        np.testing.assert_array_equal(kio.read_pgm(ref), exp[f"img{depth}"])
        out = tmp_path / f"img{depth}.pgm"
        kio.write_pgm(out, exp["img"], depth)
        assert _bytes(out) == _bytes(ref)
    np.testing.assert_array_equal(kio.read_pgm(os.path.join(IOD, "comment.pgm")), exp["comment"])


def test_config_and_json(tmp_path):
    from paper_2410_00233_b200 import io as kio

    with open(os.path.join(IOD, "opts.json")) as fh:
        assert kio.read_config(os.path.join(IOD, "opts.cfg")) == json.load(fh)
    out = tmp_path / "payload.json"
    kio.write_json(out, {"a": [1.5, float("inf"), float("nan")], "b": np.int64(3), "c": {"d": -float("inf")},
                         "e": np.arange(3)})
    assert _bytes(out) == _bytes(os.path.join(IOD, "payload.json"))


def test_kron_dir_metadata_and_terms():
    from paper_2410_00233_b200 import io as kio

    with open(os.path.join(IOD, "kron", "meta.json")) as fh:
        meta = json.load(fh)
    assert meta["k"] == 2 and meta["scheme"] == {"m1": 3, "m2": 4, "n1": 2, "n2": 5}
    assert kio.read_mtx(os.path.join(IOD, "kron", "ax_1.mtx")).shape == (3, 2)
    assert kio.read_mtx(os.path.join(IOD, "kron", "ay_2.mtx")).shape == (4, 5)


def test_errors(tmp_path):
    from paper_2410_00233_b200 import ValidationError
    from paper_2410_00233_b200 import io as kio

    bad = tmp_path / "bad.mtx"
    bad.write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(ValidationError):
        kio.read_mtx(bad)
    trunc = tmp_path / "trunc.mtx"
    trunc.write_bytes(_bytes(os.path.join(IOD, "m64.mtx"))[:-8])
    with pytest.raises(ValidationError):
        kio.read_mtx(trunc)
    with pytest.raises(ValidationError):
        kio.write_mtx(tmp_path / "i.mtx", np.ones((2, 2), dtype=np.int32))
    with pytest.raises(ValidationError):
        kio.write_pgm(tmp_path / "x.pgm", np.ones((2, 2)), depth=12)
    cfg = tmp_path / "c.cfg"
    cfg.write_text("novalue\n")
    with pytest.raises(ValidationError):
        kio.read_config(cfg)


def test_cli_parser_and_option_merging(tmp_path):
    """Option tables / config merging (cli.py:200-225) -- no device needed."""
    from paper_2410_00233_b200 import cli

    cfg = tmp_path / "o.cfg"
    cfg.write_text("k-max = 12\nprec = single\nsparse = yes\n")
    ns = cli.build_parser().parse_args(["approx", "--config", str(cfg), "--k-max", "7", "--out-dir", "x"])
    v = cli.resolve_options(cli._APPROX, ns)
    assert (v["k_max"], v["prec"], v["sparse"], v["p"], v["out_dir"]) == (7, "single", True, 2, "x")
    cfg.write_text("bogus = 1\n")
    ns = cli.build_parser().parse_args(["approx", "--config", str(cfg)])
    assert cli.main(["approx", "--config", str(cfg)]) == 2
    assert cli.main(["approx", "--out-dir", str(tmp_path / "o"), "--psf", "x.mtx"]) == 2      # no --side
    assert cli.main(["deblur", "--out-dir", str(tmp_path / "d"), "--observed", str(tmp_path / "missing.pgm"),
                     "--matrix", "m.mtx", "--beta", "0.1"]) == 4
