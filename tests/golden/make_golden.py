"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py [reflexive|sparse]

(``reflexive`` / ``sparse`` / ``cli`` regenerate only ra_reflexive.npz /
ra_sparse.npz / the io+cli file fixtures under tests/golden/io and tests/golden/cli.)

Writes ``tests/golden/*.npz``.  Every array in them is an input or an output
of the unmodified reference package ``kronblur`` (``pkg/src/kronblur``); the
oracle (``oracle/``) and the CUDA path are checked against these files, which
travel to the GPU box (the reference itself does not).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from kronblur.blurmodel import Psf, build_blur_matrix, make_test_image  # noqa: E402
from kronblur.cgls import CglsConfig, cgls_solve  # noqa: E402
from kronblur.exceptions import RankDeficiencyError  # noqa: E402
from kronblur.kronop import assemble  # noqa: E402
from kronblur.linalg import cast, orthonormalize, svd_small, vec  # noqa: E402
from kronblur.lowrank import EgkbConfig, RsvdConfig, egkb, rsvd  # noqa: E402
from kronblur.rearrange import BlockScheme, rearrange  # noqa: E402
from kronblur.splitbregman import SbConfig, sb_run  # noqa: E402

from paper_2410_00233_b200 import datagen  # noqa: E402


def spectral_matrix(rng, m, n, sigmas):
    """Same construction as the reference's tests/conftest.py:45-51."""
    sigmas = np.asarray(sigmas, dtype=np.float64)
    r = sigmas.size
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (u * sigmas) @ v.T


def geometric(count, ratio=2.0):
    return ratio ** (-np.arange(count, dtype=np.float64))


def trace_dict(tr):
    return dict(alphas=np.array(tr.alphas), ts=np.array(tr.ts), zetas=np.array(tr.zetas),
                nus=np.array(tr.nus), chosen_k=tr.chosen_k, k_p=tr.k_p,
                stop_reason=tr.stop_reason, breakdown=tr.breakdown)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def egkb_case(prefix, b_mat, cfg_kwargs, out, y0=None):
    svd, tr = egkb(b_mat, EgkbConfig(**cfg_kwargs), y0=y0)
    out[prefix + "u"] = svd.u
    out[prefix + "sigma"] = svd.sigma
    out[prefix + "v"] = svd.v
    for k, v in trace_dict(tr).items():
        out[prefix + "tr_" + k] = np.asarray(v)
    out[prefix + "cfg"] = np.asarray(json.dumps(cfg_kwargs))


def main():
    rng = np.random.default_rng(12345)

    # 1. structured R(A) closed form vs the reference's dense rearrange(build_blur_matrix)
    ra = {}
    for i, (kh, kw, n) in enumerate([(3, 5, 7), (5, 3, 6), (9, 9, 10), (1, 3, 6), (7, 7, 12)]):
        psf = Psf(rng.random((kh, kw)))
        r_mat = rearrange(build_blur_matrix(psf, n), BlockScheme.square_image(n))
        q = rng.standard_normal(n * n)
        s = rng.standard_normal(n * n)
        ra[f"c{i}_psf"] = psf.kernel
        ra[f"c{i}_n"] = n
        ra[f"c{i}_q"] = q
        ra[f"c{i}_s"] = s
        ra[f"c{i}_Rq"] = r_mat @ q
        ra[f"c{i}_RTs"] = r_mat.T @ s
        ra[f"c{i}_sigma"] = np.linalg.svd(r_mat, compute_uv=False)
    # padded even PSF (SURVEY §7 hard part 4) with the config generator, n=16
    n = 16
    kpad = datagen.rotated_gaussian_psf(n)
    psf = Psf(kpad)
    a_mat = build_blur_matrix(psf, n)
    r_mat = rearrange(a_mat, BlockScheme.square_image(n))
    q = rng.standard_normal(n * n)
    s = rng.standard_normal(n * n)
    x_img = datagen.cartoon_image(n)
    ra.update(pad_psf=psf.kernel, pad_n=n, pad_q=q, pad_s=s, pad_Rq=r_mat @ q,
              pad_RTs=r_mat.T @ s, pad_sigma=np.linalg.svd(r_mat, compute_uv=False),
              pad_x=vec(x_img), pad_Ax=a_mat @ vec(x_img))
    save("ra_structured", **ra)

    # 2. eGKB known-answer cases (shapes from the reference tests/test_lowrank.py)
    eg = {}
    egkb_case("diag_", np.diag([5.0, 3.0, 1.0]), dict(k_max=3, k_min=3, seed=1), eg)
    b = spectral_matrix(rng, 40, 30, geometric(5))
    eg["rank5_b"] = b
    egkb_case("rank5_", b, dict(k_max=10, p=2, tau=1e-30, seed=3), eg)
    b = spectral_matrix(rng, 50, 40, geometric(40, 1.15))
    eg["fact_b"] = b
    egkb_case("fact64_", b, dict(k_max=12, p=2, tau=1e-30, k_min=12, seed=0), eg)
    egkb_case("fact32_", cast(b, "single"), dict(k_max=12, p=2, tau=1e-30, k_min=12, seed=0), eg)
    b = spectral_matrix(rng, 40, 40, geometric(20, 8.0))
    eg["decay_b"] = b
    egkb_case("decay_", b, dict(k_max=15, p=2, tau=1e-6, seed=5), eg)
    egkb_case("decay32_", cast(b, "single"), dict(k_max=15, p=3, tau=1e-6, seed=5), eg)
    b = spectral_matrix(rng, 60, 40, geometric(20, 2.0))
    eg["accept3_b"] = b
    egkb_case("accept3_", b, dict(k_max=15, p=4, tau=2e-5, seed=1), eg)
    egkb_case("accept3s_", cast(b, "single"), dict(k_max=15, p=4, tau=2e-5, seed=1), eg)
    b = spectral_matrix(rng, 20, 15, geometric(15, 1.5))
    y0 = rng.standard_normal(20)
    eg["y0_b"] = b
    eg["y0_y0"] = y0
    egkb_case("y0_", b, dict(k_max=5, k_min=5, tau=1e-30), eg, y0=y0)
    # blur configs at small n (fp32 dense R, the reference's "SP" path)
    for name, side in (("n64", 32), ("n256", 48)):
        prob = datagen.make_problem(name, n=side)
        r32 = cast(rearrange(build_blur_matrix(Psf(prob.psf), side), BlockScheme.square_image(side)), "single")
        eg[f"blur_{name}_psf"] = prob.psf
        eg[f"blur_{name}_n"] = side
        egkb_case(f"blur_{name}_", r32, dict(prob.egkb), eg)
    save("egkb_kat", **eg)

    # 3. RSVD + orthonormalize
    rs = {}
    b = spectral_matrix(rng, 60, 50, geometric(30))
    rs["sig_b"] = b
    for tag, mat in (("d", b), ("s", cast(b, "single"))):
        svd = rsvd(mat, RsvdConfig(k=5, p=8, q=2, seed=2))
        rs[f"sig{tag}_u"], rs[f"sig{tag}_sigma"], rs[f"sig{tag}_v"] = svd.u, svd.sigma, svd.v
    b = spectral_matrix(rng, 30, 80, geometric(20))
    rs["wide_b"] = b
    svd = rsvd(b, RsvdConfig(k=4, p=6, q=2, seed=3))
    rs["wide_u"], rs["wide_sigma"], rs["wide_v"] = svd.u, svd.sigma, svd.v
    b = spectral_matrix(rng, 20, 15, [3.0, 1.0])
    rs["rankdef_b"] = b
    try:
        rsvd(b, RsvdConfig(k=4, p=2, q=1, seed=5))
        rs["rankdef_col"] = -1
    except RankDeficiencyError as err:
        rs["rankdef_col"] = err.column
    m = rng.standard_normal((50, 8))
    rs["orth_in"] = m
    rs["orth_out"] = orthonormalize(m)
    rs["orth32_out"] = orthonormalize(cast(m, "single"))
    save("rsvd_kat", **rs)

    # 4. CGLS on small dense systems
    cg = {}
    for i in range(4):
        a = rng.standard_normal((30, 10))
        bb = rng.standard_normal(30)
        res = cgls_solve(a, bb, CglsConfig(i_max=40, tau=1e-6 if i % 2 else 0.0))
        cg[f"c{i}_a"], cg[f"c{i}_b"], cg[f"c{i}_x"] = a, bb, res.x
        cg[f"c{i}_iters"], cg[f"c{i}_stop"] = res.iters, res.stop
        cg[f"c{i}_rc"], cg[f"c{i}_res"] = np.array(res.rc_history), np.array(res.resnorms)
    save("cgls_kat", **cg)

    # 5. split Bregman: interchange case (test_splitbregman.py:147-162) and blur configs
    sbd = {}
    n = 8
    a = build_blur_matrix(Psf(rng.random((3, 3)) + 0.05), n)
    svd = svd_small(rearrange(a, BlockScheme.square_image(n)))
    op = assemble(svd, BlockScheme.square_image(n))
    bb = a @ vec(make_test_image(n))
    cfg = SbConfig(lam=0.1, beta=0.005, tau=0.0, l_max=5, cgls=CglsConfig(i_max=12, tau=0.0))
    sbd["inter_a"], sbd["inter_b"] = a, bb
    sbd["inter_ax"], sbd["inter_ay"] = np.stack(op.ax), np.stack(op.ay)
    sbd["inter_dense_x"] = sb_run(a, bb, cfg).x
    sbd["inter_kron_x"] = sb_run(op, bb, cfg).x

    for name, side, variants in (("n64", 32, ("anisotropic", "isotropic")),):
        prob = datagen.make_problem(name, n=side)
        r32 = cast(rearrange(build_blur_matrix(Psf(prob.psf), side), BlockScheme.square_image(side)), "single")
        svd, _ = egkb(r32, EgkbConfig(**prob.egkb))
        op = assemble(svd, BlockScheme.square_image(side))
        sbd[f"{name}_ax"], sbd[f"{name}_ay"] = np.stack(op.ax), np.stack(op.ay)
        sbd[f"{name}_b"], sbd[f"{name}_xtrue"] = prob.b, prob.x_true
        for variant in variants:
            # short protocol: the strict 1e-9 bar
            short = SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant=variant, tau=0.0, l_max=5,
                             cgls=CglsConfig(i_max=20, tau=0.0))
            res = sb_run(op, prob.b, short, x_true=prob.x_true)
            sbd[f"{name}_{variant}_short_x"] = res.x
            sbd[f"{name}_{variant}_short_re"] = np.array(res.re_history)
            # configured protocol, truncated to 10 outer sweeps
            full = SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant=variant, tau=0.0, l_max=10,
                            cgls=CglsConfig(i_max=100, tau=1e-4))
            res = sb_run(op, prob.b, full, x_true=prob.x_true)
            sbd[f"{name}_{variant}_cfg_x"] = res.x
            sbd[f"{name}_{variant}_cfg_iters"] = np.array(res.cgls_iters)
            sbd[f"{name}_{variant}_cfg_rc"] = np.array(res.rc_history)
            sbd[f"{name}_{variant}_cfg_re"] = np.array(res.re_history)
            sbd[f"{name}_{variant}_cfg_isnr"] = np.array(res.isnr_history)
    save("sb_kat", **sbd)

    # 6. configs[0] at full size (n=64): reference eGKB on the dense fp32 R(A)
    prob = datagen.make_problem("n64")
    a_mat = build_blur_matrix(Psf(prob.psf), 64)
    r32 = cast(rearrange(a_mat, BlockScheme.square_image(64)), "single")
    cf = {"psf": prob.psf, "b": prob.b, "x_true": prob.x_true, "Ax_true": a_mat @ prob.x_true}
    svd, tr = egkb(r32, EgkbConfig(**prob.egkb))
    cf.update(u=svd.u, sigma=svd.sigma, v=svd.v)
    for k, v in trace_dict(tr).items():
        cf["tr_" + k] = np.asarray(v)
    svd_auto, tr_auto = egkb(r32, EgkbConfig(k_max=20))
    cf.update(auto_sigma=svd_auto.sigma, auto_chosen=tr_auto.chosen_k, auto_kp=tr_auto.k_p,
              auto_reason=tr_auto.stop_reason, auto_nus=np.array(tr_auto.nus))
    op = assemble(svd, BlockScheme.square_image(64))
    short = SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant="anisotropic", tau=0.0, l_max=5,
                     cgls=CglsConfig(i_max=20, tau=0.0))
    cf["sb_short_x"] = sb_run(op, prob.b, short).x
    save("config_n64", **cf)


def reflexive():
    """Reflexive-BC R(A) (blurmodel.py:80-84, 122-126): dense reference R, products,
    singular values, and fp32 eGKB runs on the dense reference R."""
    rng = np.random.default_rng(2024)
    rf = {}
    cases = [(3, 5, 7), (5, 3, 6), (9, 9, 10), (1, 3, 6), (13, 13, 7), (11, 3, 12)]
    for i, (kh, kw, n) in enumerate(cases):
        psf = Psf(rng.random((kh, kw)))
        r_mat = rearrange(build_blur_matrix(psf, n, bc="reflexive"), BlockScheme.square_image(n))
        q = rng.standard_normal(n * n)
        s = rng.standard_normal(n * n)
        rf[f"c{i}_psf"] = psf.kernel
        rf[f"c{i}_n"] = n
        rf[f"c{i}_R"] = r_mat
        rf[f"c{i}_q"] = q
        rf[f"c{i}_s"] = s
        rf[f"c{i}_Rq"] = r_mat @ q
        rf[f"c{i}_RTs"] = r_mat.T @ s
        rf[f"c{i}_sigma"] = np.linalg.svd(r_mat, compute_uv=False)
    rf["ncases"] = len(cases)
    # config generators at small sides, fp32 dense R (the reference's SP path)
    for name, side in (("n64", 32), ("n256", 40)):
        prob = datagen.make_problem(name, n=side)
        r32 = cast(rearrange(build_blur_matrix(Psf(prob.psf), side, bc="reflexive"),
                             BlockScheme.square_image(side)), "single")
        rf[f"blur_{name}_psf"] = prob.psf
        rf[f"blur_{name}_n"] = side
        egkb_case(f"blur_{name}_", r32, dict(prob.egkb), rf)
    save("ra_reflexive", **rf)


def sparse():
    """R(A) of unstructured sparse A (rearrange.py:67-75) and the reference engines on it."""
    rng = np.random.default_rng(31337)
    sp = {}
    # 1. random sparse A, non-square block scheme
    scheme = BlockScheme(6, 5, 4, 7)
    a = rng.standard_normal(scheme.shape) * (rng.random(scheme.shape) < 0.12)
    sp["s1_a"], sp["s1_scheme"] = a, np.array([6, 5, 4, 7])
    r = rearrange(a, scheme)
    sp["s1_R"] = r
    for tag, mat in (("d", r), ("s", cast(r, "single"))):
        cfg = dict(k_max=6, p=2, tau=1e-30, k_min=6, seed=4)
        egkb_case(f"s1{tag}_", mat, cfg, sp)
    svd = rsvd(r, RsvdConfig(k=4, p=3, q=2, seed=6))
    sp["s1_rsvd_sigma"], sp["s1_rsvd_u"], sp["s1_rsvd_v"] = svd.sigma, svd.u, svd.v
    # 2. spatially variant blur: PSF blur + sparse random couplings, n = 16
    n = 16
    a = build_blur_matrix(Psf(rng.random((5, 5))), n)
    extra = (rng.random(a.shape) < 0.002) * rng.random(a.shape) * 0.05
    a = a + extra
    sp["s2_a"], sp["s2_n"] = a, n
    r = rearrange(a, BlockScheme.square_image(n))
    sp["s2_R"] = r
    egkb_case("s2s_", cast(r, "single"), dict(k_max=12, tau=1e-4), sp)
    egkb_case("s2d_", r, dict(k_max=8, k_min=8, p=2, tau=1e300), sp)
    save("ra_sparse", **sp)


def cli_io():
    """File formats written by the reference's io.py, and reference CLI runs
    (approx -> deblur -> sweep) on a small PSF problem, for the f4 parity tests."""
    import shutil

    from kronblur import io as rio
    from kronblur.cli import main as ref_cli
    from kronblur.kronop import KroneckerSum

    rng = np.random.default_rng(777)
    iod = os.path.join(HERE, "io")
    shutil.rmtree(iod, ignore_errors=True)
    os.makedirs(iod)
    with open(os.path.join(iod, "opts.cfg"), "w") as fh:
        fh.write("# defaults\nk-max = 12   # cap\n\nprec=single\n tau-egkb = 1e-6\n")
    m64, m32, v6 = rng.standard_normal((5, 7)), rng.standard_normal((3, 4)).astype(np.float32), rng.standard_normal(6)
    rio.write_mtx(os.path.join(iod, "m64.mtx"), m64)
    rio.write_mtx(os.path.join(iod, "m32.mtx"), m32)
    rio.write_mtx(os.path.join(iod, "vec.mtx"), v6)
    img = rng.random((9, 11))
    img[0, 0], img[1, 1] = -0.2, 1.3           # clipped
    rio.write_pgm(os.path.join(iod, "img8.pgm"), img, 8)
    rio.write_pgm(os.path.join(iod, "img16.pgm"), img, 16)
    with open(os.path.join(iod, "comment.pgm"), "wb") as fh:   # header comments are legal PGM
        fh.write(b"P5\n# made by hand\n3 2\n# depth\n255\n" + bytes([0, 128, 255, 1, 2, 3]))
    np.savez(os.path.join(iod, "expected.npz"), m64=m64, m32=m32, vec=v6, img=img,
             img8=rio.read_pgm(os.path.join(iod, "img8.pgm")), img16=rio.read_pgm(os.path.join(iod, "img16.pgm")),
             comment=rio.read_pgm(os.path.join(iod, "comment.pgm")))
    with open(os.path.join(iod, "opts.json"), "w") as fh:   # what the reference's read_config returns
        json.dump(rio.read_config(os.path.join(iod, "opts.cfg")), fh)
    op = KroneckerSum([rng.standard_normal((3, 2)) for _ in range(2)], [rng.standard_normal((4, 5)) for _ in range(2)],
                      BlockScheme(3, 4, 2, 5))
    rio.save_kron_dir(op, os.path.join(iod, "kron"), extra_meta={"engine": "egkb", "k_p": 4, "rho": 1.0})
    rio.write_json(os.path.join(iod, "payload.json"), {"a": [1.5, float("inf"), float("nan")], "b": np.int64(3),
                                                     "c": {"d": -float("inf")}, "e": np.arange(3)})

    # reference CLI: simulate inputs are made here (numpy), then approx / deblur / sweep
    cli = os.path.join(HERE, "cli")
    shutil.rmtree(cli, ignore_errors=True)
    os.makedirs(cli)
    n = 16
    psf = Psf(np.pad(rng.random((5, 5)) + 0.1, ((0, 0), (0, 0))))
    rio.write_mtx(os.path.join(cli, "psf.mtx"), psf.kernel)
    x_img = make_test_image(n)
    a = build_blur_matrix(psf, n)
    b = a @ vec(x_img)
    b = b + 0.002 * np.random.default_rng(3).standard_normal(b.shape)
    rio.write_pgm(os.path.join(cli, "observed.pgm"), b.reshape(n, n, order="F"), 16)
    rio.write_pgm(os.path.join(cli, "truth.pgm"), x_img, 16)
    rio.write_mtx(os.path.join(cli, "matrix.mtx"), a)
    runs = {
        "approx_single": ["approx", "--psf", "psf.mtx", "--side", str(n), "--prec", "single", "--k-max", "10"],
        "approx_double": ["approx", "--psf", "psf.mtx", "--side", str(n), "--k-max", "8", "--k-min", "8",
                          "--tau-egkb", "1e300"],
        "approx_rsvd": ["approx", "--matrix", "matrix.mtx", "--engine", "rsvd", "--k", "3", "--p", "1", "--q", "2"],
    }
    cwd = os.getcwd()
    os.chdir(cli)
    try:
        for name, argv in runs.items():
            assert ref_cli(argv + ["--out-dir", name]) == 0, name
        assert ref_cli(["deblur", "--operator-dir", "approx_double/operator", "--observed", "observed.pgm",
                        "--truth", "truth.pgm", "--lam", "0.1", "--gamma", "2.0", "--l-max", "5", "--tau-sb", "0",
                        "--i-max", "20", "--tau-cgls", "0", "--out-dir", "deblur"]) == 0
        assert ref_cli(["sweep", "--operator-dir", "approx_double/operator", "--observed", "observed.pgm",
                        "--truth", "truth.pgm", "--count", "4", "--lam-min", "0.02", "--lam-max", "0.5",
                        "--l-max", "3", "--tau-sb", "0", "--i-max", "20", "--tau-cgls", "0", "--out-dir", "sweep"]) == 0
        assert ref_cli(["approx", "--psf", "psf.mtx", "--side", "0", "--out-dir", "bad"]) == 2
    finally:
        os.chdir(cwd)
    shutil.rmtree(os.path.join(cli, "bad"), ignore_errors=True)
    print("wrote", iod, cli)


if __name__ == "__main__":
    if sys.argv[1:] == ["cli"]:
        cli_io()
    elif sys.argv[1:] == ["reflexive"]:
        reflexive()
    elif sys.argv[1:] == ["sparse"]:
        sparse()
    else:
        main()
        reflexive()
        sparse()
        cli_io()
