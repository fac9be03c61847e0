"""`gkpca pca` front end (gkpca.cpp:170-308): options, output artifacts
(singvals.csv, U.gmx, V.gmx, stats.json, manifest.json) and exit codes."""
import json
import os

import numpy as np
import pytest

from conftest import principal_angles, rel_err, sigma_rel_err


def _bed(tmp_path, p=120, n=90, seed=0, missing=0.03):
    from paper_1808_03374_b200 import genio
    rng = np.random.default_rng(seed)
    # two populations so the spectrum has structure
    f = rng.uniform(0.1, 0.9, size=p)
    pop = np.arange(n) % 2
    fp = np.clip(f[:, None] + np.where(pop[None, :] == 0, 0.15, -0.15), 0.02, 0.98)
    d = rng.binomial(2, fp).astype(np.uint8)
    d[rng.random((p, n)) < missing] = 3
    pre = str(tmp_path / "geno")
    genio.write_bed(genio.encode(d), p, n, pre + ".bed", pre + ".bim", pre + ".fam")
    return pre, d


def run(argv):
    from paper_1808_03374_b200 import cli
    return cli.main(argv)


# ---------------------------------------------------------------- CPU
def test_usage_errors_exit_4(capsys):
    assert run([]) == 4
    assert run(["pca"]) == 4                                    # missing input
    assert run(["pca", "x.bed", "--standardize", "bogus"]) == 4
    assert run(["pca", "x.bed", "--reorth", "sometimes"]) == 4
    assert run(["nope"]) == 4


def test_unsupported_input_exit_3(tmp_path, capsys):
    p = tmp_path / "m.txt"
    p.write_text("1,2\n")
    assert run(["pca", str(p), "--out", str(tmp_path / "o")]) == 3
    assert "unsupported input format (expect .gmx or .bed)" in capsys.readouterr().err


def test_bad_bed_exit_3(tmp_path, capsys):
    pre, _ = _bed(tmp_path, 8, 8)
    with open(pre + ".bed", "r+b") as f:
        f.write(b"\x00")
    assert run(["pca", pre + ".bed", "--out", str(tmp_path / "o")]) == 3
    assert "bad magic" in capsys.readouterr().err


def test_gmx_and_csv_writers(tmp_path):
    from paper_1808_03374_b200 import genio
    M = np.arange(12, dtype=float).reshape(3, 4) / 7.0
    genio.write_dense(str(tmp_path / "a.gmx"), M)
    raw = (tmp_path / "a.gmx").read_bytes()
    assert raw[:4] == b"GMX1" and len(raw) == 16 + 12 * 8
    assert np.frombuffer(raw[4:16], dtype="<u4").tolist() == [3, 4, 0]
    assert np.array_equal(np.frombuffer(raw[16:], dtype="<f8"), M.ravel(order="F"))
    assert np.array_equal(genio.read_dense(str(tmp_path / "a.gmx")), M)
    genio.write_csv_matrix(str(tmp_path / "s.csv"), np.array([1.0, 1 / 3, 1e-300]))
    assert (tmp_path / "s.csv").read_text() == \
        "c1\n1\n0.33333333333333331\n1e-300\n"
    (tmp_path / "bad.gmx").write_bytes(b"GMX1" + bytes(12) + b"x")
    with pytest.raises(Exception, match="payload size mismatch"):
        genio.read_dense(str(tmp_path / "bad.gmx"))


def test_make_gkl_options_defaults():
    from paper_1808_03374_b200 import cli
    a = cli.build_parser().parse_args(["pca", "x.bed", "-k", "7", "--restart", "thick"])
    o = cli.make_gkl_options(a, 1000)
    assert (o.max_subspace, o.keep, o.record_history) == (20, 10, True)   # max(2k,20), max(k, D/2)
    o = cli.make_gkl_options(a, 15)
    assert (o.max_subspace, o.keep) == (15, 7)                            # capped by min(m, n)


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("standardize,scheme", [("none", 3), ("unit", 0), ("binomial", 1),
                                                ("hwe", 2)])
def test_pca_bed_end_to_end(gkb, orc, tmp_path, standardize, scheme):
    from paper_1808_03374_b200 import cli, genio
    pre, _ = _bed(tmp_path)
    out = tmp_path / f"out_{standardize}"
    argv = ["pca", pre + ".bed", "-k", "5", "--tol", "1e-10", "--standardize", standardize,
            "--restart", "thick", "--out", str(out), "--seed", "3"]
    assert run(argv) == 0
    names = sorted(os.listdir(out))
    assert names == ["U.gmx", "V.gmx", "manifest.json", "singvals.csv", "stats.json"]
    sv = np.loadtxt(out / "singvals.csv", delimiter=",", skiprows=1)
    U, V = genio.read_dense(str(out / "U.gmx")), genio.read_dense(str(out / "V.gmx"))
    assert U.shape == (120, 5) and V.shape == (90, 5)
    stats = json.loads((out / "stats.json").read_text())
    assert stats["algorithm"] == "gkl" and stats["converged"] and not stats["partial_results"]
    assert len(stats["ritz_history"]) == len(stats["err_history"]) > 0
    man = json.loads((out / "manifest.json").read_text())
    assert man["command"] == "pca" and man["seed"] == 3 and man["config"]["k"] == 5
    # oracle: same payload, same scaling, same options
    payload, p, n = genio.read_bed(pre + ".bed", pre + ".bim", pre + ".fam")
    mu, inv_s = orc.marker_scaling(orc.marker_counts(payload, p, n), n, scheme)
    ref = orc.GenoOracle(payload, p, n, mu, inv_s)
    a = cli.build_parser().parse_args(argv)
    o = orc.svdl(ref, orc.Options.from_gkl(cli.make_gkl_options(a, min(p, n))))
    assert sigma_rel_err(sv, o.singvals) <= 1e-9
    assert principal_angles(U, o.U) < 1e-6 and principal_angles(V, o.V) < 1e-6
    # a rerun writes byte-identical artifacts (no timestamps; wall time only in stats)
    out2 = tmp_path / f"out2_{standardize}"
    argv[argv.index("--out") + 1] = str(out2)
    assert run(argv) == 0
    for f in ("singvals.csv", "U.gmx", "V.gmx", "manifest.json"):
        assert (out / f).read_bytes() == (out2 / f).read_bytes(), f


@pytest.mark.gpu
def test_pca_unconverged_exit_2(gkb, tmp_path, capsys):
    pre, _ = _bed(tmp_path)
    out = tmp_path / "o"
    assert run(["pca", pre + ".bed", "-k", "5", "--max-mvps", "6", "--out", str(out)]) == 2
    assert "not converged within budget" in capsys.readouterr().err
    assert json.loads((out / "stats.json").read_text())["partial_results"] is True
    assert (out / "singvals.csv").exists()


@pytest.mark.gpu
def test_pca_gmx_input(gkb, tmp_path):
    from paper_1808_03374_b200 import genio
    rng = np.random.default_rng(2)
    X = rng.standard_normal((60, 4)) @ rng.standard_normal((4, 50)) + 0.01 * rng.standard_normal((60, 50))
    genio.write_dense(str(tmp_path / "x.gmx"), X)
    out = tmp_path / "o"
    assert run(["pca", str(tmp_path / "x.gmx"), "-k", "3", "--tol", "1e-10", "--out", str(out)]) == 0
    sv = np.loadtxt(out / "singvals.csv", delimiter=",", skiprows=1)
    assert rel_err(sv, np.linalg.svd(X, compute_uv=False)[:3]) <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["qr", "normalize"])
def test_pca_subspace(gkb, tmp_path, variant):
    """--algo subspace (gkpca.cpp:251-279): singular values from the block
    iteration, V = X^T U / sigma, subspace stats keys."""
    from paper_1808_03374_b200 import genio
    pre, d = _bed(tmp_path)
    out = tmp_path / f"s_{variant}"
    rc = run(["pca", pre + ".bed", "--algo", "subspace", "--variant", variant, "-k", "3",
              "--tol", "1e-10", "--max-iters", "400", "--standardize", "unit", "--out", str(out)])
    stats = json.loads((out / "stats.json").read_text())
    assert stats["algorithm"] == "subspace" and stats["variant"] == variant
    assert set(stats) >= {"mvps", "iterations", "converged", "rank_deficient", "wall_seconds",
                          "delta_history", "invcond_history", "partial_results"}
    assert rc == (0 if stats["converged"] else 2)
    sv = np.loadtxt(out / "singvals.csv", delimiter=",", skiprows=1)
    U, V = genio.read_dense(str(out / "U.gmx")), genio.read_dense(str(out / "V.gmx"))
    # dense reference: the operator's own matrix (X = op applied to the identity)
    op = gkb.GenotypeOperator.from_bed_file(pre, scheme=gkb.ScalingScheme.kUnitVariance)
    M = op.apply_block(np.eye(op.cols()))
    ref = np.linalg.svd(M, compute_uv=False)[:3]
    if variant == "qr":
        assert rel_err(sv, ref) <= 1e-9
    else:  # the normalize variant's bar (test_subspace.cpp:139-142): top value to 1e-4 sigma_1
        assert abs(sv[0] - ref[0]) <= 1e-4 * ref[0]
    assert np.allclose(M.T @ U[:, 0] / sv[0], V[:, 0], atol=1e-10)


def test_read_csv_matrix(tmp_path):
    from paper_1808_03374_b200 import genio
    p = tmp_path / "a.csv"
    p.write_text("y\n1.5\n2\n\n-3e-2\r\n")
    assert genio.read_csv_matrix(str(p)).ravel().tolist() == [1.5, 2.0, -0.03]
    p.write_text("1,2\n3\n")
    with pytest.raises(Exception, match="ragged rows"):
        genio.read_csv_matrix(str(p))
    p.write_text("a\nb\n")
    with pytest.raises(Exception, match="non-numeric cell outside header"):
        genio.read_csv_matrix(str(p))
    p.write_text("h\n")
    with pytest.raises(Exception, match="no data rows"):
        genio.read_csv_matrix(str(p))


def test_regress_bad_pheno_exit_3(tmp_path, capsys):
    pre, _ = _bed(tmp_path, 8, 8)
    ph = tmp_path / "ph.csv"
    ph.write_text("a,b\n1,2\n")
    assert run(["regress", pre + ".bed", "--pheno", str(ph), "--out", str(tmp_path / "o")]) in (3, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 2])
def test_regress_end_to_end(gkb, tmp_path, k):
    """gkpca regress: per-marker scan entries vs the reference loop on the
    operator's dense matrix; design mode; manifest."""
    from paper_1808_03374_b200 import regress as R
    pre, d = _bed(tmp_path)
    n = d.shape[1]
    rng = np.random.default_rng(4)
    y = rng.standard_normal(n)
    ph = tmp_path / "ph.csv"
    ph.write_text("y\n" + "\n".join("%.17g" % v for v in y) + "\n")
    out = tmp_path / f"r{k}"
    rc = run(["regress", pre + ".bed", "--pheno", str(ph), "-k", str(k), "--tol", "1e-10",
              "--standardize", "unit", "--out", str(out)])
    assert rc == 0
    res = json.loads((out / "regression.json").read_text())
    assert res["mode"] == "per-marker" and res["k"] == k and res["pca_converged"]
    op = gkb.GenotypeOperator.from_bed_file(pre, scheme=gkb.ScalingScheme.kUnitVariance)
    M = op.apply_block(np.eye(n))
    Z = np.zeros((n, 0))
    if k:
        Z = gkb.svdl(op, gkb.GklOptions(k=k, tol=1e-10)).V
    for i in (0, 7, 33, 101):
        X = np.column_stack([np.ones(n), M[i]])
        f = R.pc_adjusted_fit(X, Z, y) if k else R.ols_fit(X, y)
        e = res["markers"][i]
        assert e["marker"] == i
        assert abs(e["beta"] - f.beta_hat[1]) <= 1e-8 * max(1, abs(f.beta_hat[1]))
        assert abs(e["se"] - np.sqrt(f.cov_beta[1, 1])) <= 1e-8 * np.sqrt(f.cov_beta[1, 1])
    man = json.loads((out / "manifest.json").read_text())
    assert man["command"] == "regress" and man["config"]["k"] == k
    # design mode
    dz = tmp_path / "design.csv"
    Xd = np.column_stack([np.ones(n), rng.standard_normal(n)])
    dz.write_text("\n".join(",".join("%.17g" % v for v in row) for row in Xd) + "\n")
    out2 = tmp_path / f"d{k}"
    assert run(["regress", pre + ".bed", "--pheno", str(ph), "--design", str(dz), "-k", str(k),
                "--tol", "1e-10", "--standardize", "unit", "--out", str(out2)]) == 0
    fit = json.loads((out2 / "regression.json").read_text())["fit"]
    ref = R.pc_adjusted_fit(Xd, Z, y) if k else R.ols_fit(Xd, y)
    assert np.allclose(fit["beta"], ref.beta_hat, rtol=1e-8, atol=1e-12)


# ---------------------------------------------------------------- bench
def test_bench_usage_exit_4(tmp_path, capsys):
    assert run(["bench", "x.bed"]) == 4                         # --seed is required
    assert run(["bench", "x.bed", "--seed", "1", "--standardize", "bogus"]) == 4


@pytest.mark.gpu
def test_bench_end_to_end(gkb, tmp_path, capsys):
    """gkpca bench (gkpca.cpp:424-536): every solver on one operator, mvps
    equal to the operator's own counter, errors against the dense SVD."""
    pre, _ = _bed(tmp_path, 150, 100, seed=3)
    out = tmp_path / "b"
    algos = ",".join(["gkl-pro-nr", "gkl-fro-nr", "gkl-pro-tr", "gkl-fro-tr", "subspace-qr",
                      "subspace-normalize"])
    assert run(["bench", pre + ".bed", "--seed", "5", "-k", "4", "--tol", "1e-10",
                "--algos", algos, "--standardize", "unit", "--out", str(out)]) == 0
    lines = (out / "bench.csv").read_text().splitlines()
    assert lines[0] == "algorithm,mvps,seconds,l1_err,rel_err_k"
    rows = [ln.split(",") for ln in lines[1:]]
    assert [r[0] for r in rows] == algos.split(",")
    for name, mv, sec, l1, rel in rows:
        assert int(mv) > 0 and float(sec) > 0.0
        assert np.isfinite(float(l1)) and np.isfinite(float(rel))
        if name == "subspace-normalize":  # the paper's naive variant: no re-orthogonalization,
            continue                      # trailing values collapse onto the leading one
        tol = 1e-8 if name.startswith("gkl") else 1e-4
        assert float(l1) < tol and float(rel) < tol, (name, l1, rel)
    man = json.loads((out / "manifest.json").read_text())
    assert man["command"] == "bench" and man["seed"] == 5 and man["config"]["k"] == 4
    # above the oracle cap the error columns are nan and a note goes to stderr
    assert run(["bench", pre + ".bed", "--seed", "5", "-k", "3", "--algos", "gkl-pro-nr",
                "--oracle-cap", "10", "--out", str(out)]) == 0
    assert "dense oracle skipped" in capsys.readouterr().err
    row = (out / "bench.csv").read_text().splitlines()[1].split(",")
    assert row[3] == "nan" and row[4] == "nan"
    assert run(["bench", pre + ".bed", "--seed", "5", "--algos", "gkl-xx", "--out",
                str(out)]) == 4


def test_impute_mean_and_orthonormality_error():
    """genio.impute_mean (genio.cpp:124-148) against the oracle's decode/impute
    semantics, and orthonormality_error (orth.cpp:23-29)."""
    from paper_1808_03374_b200 import genio
    from paper_1808_03374_b200.subspace import orthonormality_error
    d = np.array([[0, 1, 3, 2], [3, 3, 3, 3], [2, 3, 2, 2]], dtype=np.uint8)
    X, allm = genio.impute_mean(d, return_all_missing=True)
    assert np.array_equal(X, [[0, 1, 1, 2], [0, 0, 0, 0], [2, 2, 2, 2]])
    assert allm.tolist() == [False, True, False]
    Q = np.linalg.qr(np.random.default_rng(0).standard_normal((20, 4)))[0]
    assert orthonormality_error(Q) <= 1e-14
    assert abs(orthonormality_error(2 * Q) - 3.0) <= 1e-12
