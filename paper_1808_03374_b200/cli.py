"""Command-line front end of the hot path: the reference's ``gkpca pca``
(/root/reference/proj/tools/gkpca.cpp:170-308, options :706-736), ``bench``
(:384-536, options :757-780) and ``regress`` (:554-682), run on the B200
operator and driver.

    python -m paper_1808_03374_b200.cli bench INPUT --seed S [--algos LIST] [-k K] [--tol T]
        [--max-mvps N] [--max-iters N] [--oracle-cap C] [--standardize ...] [--out DIR]
    python -m paper_1808_03374_b200.cli regress INPUT --pheno CSV [--design CSV] [-k K] ...
    python -m paper_1808_03374_b200.cli pca INPUT [--algo gkl] [-k K] [--tol T]
        [--max-mvps N] [--seed S] [--standardize none|unit|binomial|hwe]
        [--out DIR] [--reorth partial|full] [--omega W] [--restart none|thick]
        [--max-subspace D] [--keep K] [--variant qr|normalize] [--max-iters N]

Same inputs (.bed with companion .bim/.fam, or GMX1 .gmx), outputs
(singvals.csv, U.gmx, V.gmx, stats.json, manifest.json; genio.cpp:203-275,
gkpca.cpp:56-74,282-301) and exit codes (0 ok, 2 not converged with partial
results written, 3 FormatError, 4 usage / invalid argument, 1 other;
gkpca.cpp:43-46,803-832). A .bed input is streamed into HBM as the packed
operator (no dense copy); `--standardize none` is the reference's mean-
imputed raw matrix (`impute_mean`, genio.cpp:124-148). `hwe` adds BASELINE's
sqrt(2f(1-f)) scaling. JSON files are written with sorted keys and 2-space
indent like nlohmann::json::dump(2).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from typing import List, Optional

import numpy as np

TOOL_VERSION = "0.1.0"
EXIT_OK, EXIT_UNCONVERGED, EXIT_FORMAT, EXIT_USAGE = 0, 2, 3, 4


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 ParseError -> kExitUsage (gkpca.cpp:809-811)
        raise UsageError(message)


def _write_json(path: str, obj) -> None:
    from ._lib import FormatError
    try:
        f = open(path, "w")
    except OSError as e:
        raise FormatError(f"cannot open {path} for writing") from e
    with f:
        f.write(json.dumps(obj, indent=2, sort_keys=True, allow_nan=False) + "\n")


def _versions():
    from . import _lib
    return {"gkpca": TOOL_VERSION, "libgkb": _lib.lib.gkb_version().decode()}


def make_gkl_options(a, minmn: int):
    """make_gkl_options (gkpca.cpp:192-212)."""
    from .gkl import GklOptions, ReorthMode, RestartMode
    o = GklOptions()
    o.k = int(a.k)
    o.tol = float(a.tol)
    o.max_mvps = int(a.max_mvps)
    o.seed = int(a.seed)
    o.record_history = True
    o.reorth = ReorthMode.kFull if a.reorth == "full" else ReorthMode.kPartial
    o.omega = float(a.omega)
    if a.restart == "thick":
        o.restart = RestartMode.kThick
        o.max_subspace = int(a.max_subspace) if a.max_subspace > 0 else max(2 * o.k, 20)
        o.max_subspace = min(o.max_subspace, minmn)
        o.keep = int(a.keep) if a.keep > 0 else max(o.k, o.max_subspace // 2)
    return o


def load_operator(path: str, standardize: str):
    """load_matrix + apply_standardize (gkpca.cpp:89-108): a .bed input becomes
    the packed device operator, a .gmx input a device DenseOperator."""
    from . import genio
    from ._lib import FormatError
    from .gkl import DenseOperator, GenotypeOperator, ScalingScheme
    ext = os.path.splitext(path)[1]
    if ext == ".bed":
        scheme = {"none": ScalingScheme.kNone, "unit": ScalingScheme.kUnitVariance,
                  "binomial": ScalingScheme.kBinomial, "hwe": ScalingScheme.kHwe}[standardize]
        base = path[:-4]
        return GenotypeOperator.from_bed_file(path, base + ".bim", base + ".fam", scheme=scheme)
    if ext == ".gmx":
        X = genio.read_dense(path)
        if standardize in ("unit", "binomial"):
            X = genio.standardize_dense(X, standardize)
        elif standardize == "hwe":
            raise ValueError("--standardize hwe applies to .bed genotype inputs")
        return DenseOperator(X)
    raise FormatError(f"{path}: unsupported input format (expect .gmx or .bed)")


def run_pca(a) -> int:
    """run_pca (gkpca.cpp:214-308)."""
    from . import genio
    from .gkl import svdl
    op = load_operator(a.input, a.standardize)
    os.makedirs(a.out, exist_ok=True)
    if a.algo == "gkl":
        opts = make_gkl_options(a, min(op.rows(), op.cols()))
        r = svdl(op, opts)
        converged = bool(r.stats.converged)

        def trim(h):  # history rows are NaN-padded to k; the reference keeps head(min(k, j))
            h = np.asarray(h, dtype=np.float64)
            return [float(v) for v in h if not math.isnan(v)]

        singvals, U, V = r.singvals, r.U, r.V
        stats = {"algorithm": "gkl", "mvps": r.stats.mvps, "steps": r.stats.steps,
                 "restarts": r.stats.restarts, "reorth_count": r.stats.reorth_count,
                 "deflations": r.stats.deflations, "converged": converged,
                 "wall_seconds": r.stats.wall_seconds,
                 "err_estimates": [float(v) for v in r.err_estimates],
                 "ritz_history": [trim(h) for h in r.stats.ritz_history],
                 "err_history": [trim(h) for h in r.stats.err_history]}
    else:  # subspace (gkpca.cpp:251-279)
        import time
        from .subspace import SubspaceVariant, subspace_iterate
        variant = SubspaceVariant.kNormalize if a.variant == "normalize" else SubspaceVariant.kQr
        t0 = time.perf_counter()
        r = subspace_iterate(op, int(a.k), variant, float(a.tol), int(a.max_iters), int(a.seed))
        wall = time.perf_counter() - t0
        singvals, U = r.singvals, r.basis
        # right vectors from the left basis: v_i = X^T u_i / sigma_i (not counted as mvps)
        V = op.apply_adjoint_block(U)
        for i in range(U.shape[1]):
            if i < singvals.size and singvals[i] > 0.0:
                V[:, i] /= singvals[i]
        converged = bool(r.converged)
        stats = {"algorithm": "subspace", "variant": a.variant, "mvps": r.mvps,
                 "iterations": r.state.iterations, "converged": converged,
                 "rank_deficient": bool(r.rank_deficient), "wall_seconds": wall,
                 "delta_history": [float(v) for v in r.state.delta_history],
                 "invcond_history": [float(v) for v in r.state.invcond_history]}
    genio.write_csv_matrix(os.path.join(a.out, "singvals.csv"), singvals)
    genio.write_dense(os.path.join(a.out, "U.gmx"), U)
    genio.write_dense(os.path.join(a.out, "V.gmx"), V)
    stats["partial_results"] = not converged
    _write_json(os.path.join(a.out, "stats.json"), stats)
    config = {"input": a.input, "algo": a.algo, "k": a.k, "tol": a.tol, "max_mvps": a.max_mvps,
              "standardize": a.standardize, "reorth": a.reorth, "omega": a.omega,
              "restart": a.restart, "max_subspace": a.max_subspace, "keep": a.keep,
              "variant": a.variant, "max_iters": a.max_iters}
    # write_manifest (gkpca.cpp:61-71): no timestamps -> reruns are byte-identical
    _write_json(os.path.join(a.out, "manifest.json"),
                {"command": "pca", "config": config, "seed": a.seed, "versions": _versions()})
    if not converged:
        sys.stderr.write("gkpca pca: not converged within budget; partial results written "
                         "(stats.json has partial_results=true)\n")
        return EXIT_UNCONVERGED
    return EXIT_OK


BENCH_ALGOS = ("gkl-pro-nr", "gkl-fro-nr", "gkl-pro-tr", "gkl-fro-tr", "subspace-qr",
               "subspace-normalize")


def _g17(x: float) -> str:  # std::snprintf("%.17g")
    return "%.17g" % x


def run_bench(a) -> int:
    """run_bench (gkpca.cpp:424-536): every listed solver on the same operator,
    mvps checked against the operator's own product counter, errors against a
    dense SVD when min(m, n) <= --oracle-cap; bench.csv + manifest.json."""
    import time
    from .gkl import GklOptions, ReorthMode, RestartMode, svdl
    from .subspace import SubspaceVariant, subspace_iterate
    algos = [t for t in a.algos.split(",") if t]  # split_csv_list (:400-413)
    op = load_operator(a.input, a.standardize)
    k = int(a.k)
    if not algos:
        raise ValueError("bench: --algos list is empty")
    for name in algos:
        if name not in BENCH_ALGOS:
            raise ValueError(f"bench: unknown algorithm '{name}'")
    m, n = op.rows(), op.cols()
    minmn = min(m, n)
    oracle = None
    if minmn <= int(a.oracle_cap):
        # the dense matrix the operator applies, through the operator itself
        M = op.apply_block(np.eye(n))
        oracle = np.linalg.svd(M, compute_uv=False)[:min(k, minmn)]
    else:
        sys.stderr.write(f"gkpca bench: dense oracle skipped (min dimension {minmn} > cap "
                         f"{a.oracle_cap}); error columns left as nan\n")
    rows = []
    for name in algos:
        before = op.mvps()
        if name.startswith("gkl"):
            o = GklOptions(k=k, tol=float(a.tol), max_mvps=int(a.max_mvps), seed=int(a.seed))
            o.reorth = ReorthMode.kFull if "fro" in name else ReorthMode.kPartial
            if "-tr" in name:
                o.restart = RestartMode.kThick
                o.max_subspace = min(max(2 * k, 20), minmn)
                o.keep = max(k, o.max_subspace // 2)
            r = svdl(op, o)
            vals, reported, seconds = r.singvals, r.stats.mvps, r.stats.wall_seconds
        else:
            variant = (SubspaceVariant.kNormalize if name == "subspace-normalize"
                       else SubspaceVariant.kQr)
            t0 = time.perf_counter()
            r = subspace_iterate(op, k, variant, float(a.tol), int(a.max_iters), int(a.seed))
            seconds = time.perf_counter() - t0
            vals, reported = r.singvals, r.mvps
        counted = op.mvps() - before
        if reported != counted:
            raise RuntimeError("bench: solver mvp count disagrees with the operator counter")
        l1 = rel = float("nan")
        if oracle is not None:
            c = min(vals.size, oracle.size)
            l1 = float(np.sum(np.abs(vals[:c] - oracle[:c])))
            if vals.size >= k and oracle.size >= k and oracle[k - 1] > 0.0:
                rel = float(abs(vals[k - 1] - oracle[k - 1]) / oracle[k - 1])
        rows.append((name, counted, seconds, l1, rel))
    os.makedirs(a.out, exist_ok=True)
    path = os.path.join(a.out, "bench.csv")
    from ._lib import FormatError
    try:
        f = open(path, "w")
    except OSError as e:
        raise FormatError(f"cannot open {path} for writing") from e
    with f:
        f.write("algorithm,mvps,seconds,l1_err,rel_err_k\n")
        for name, mv, sec, l1, rel in rows:
            f.write(f"{name},{mv},{_g17(sec)},{_g17(l1)},{_g17(rel)}\n")
    config = {"input": a.input, "algos": a.algos, "k": a.k, "tol": a.tol,
              "max_mvps": a.max_mvps, "max_iters": a.max_iters, "oracle_cap": a.oracle_cap,
              "standardize": a.standardize}
    _write_json(os.path.join(a.out, "manifest.json"),
                {"command": "bench", "config": config, "seed": a.seed, "versions": _versions()})
    return EXIT_OK


def run_regress(a) -> int:
    """run_regress (gkpca.cpp:554-680): PC-adjusted regression of a phenotype
    on every marker (device scan) or on a joint design."""
    from . import genio
    from ._lib import FormatError
    from . import regress as R
    from .gkl import DenseOperator, GklOptions, svdl
    op = load_operator(a.input, a.standardize)
    n = op.cols()
    ph = genio.read_csv_matrix(a.pheno)
    if ph.shape[1] != 1:
        raise FormatError(f"{a.pheno}: phenotype must be a single column")
    if ph.shape[0] != n:
        raise FormatError(f"{a.pheno}: phenotype rows ({ph.shape[0]}) do not match samples ({n})")
    y = ph[:, 0]
    Z = np.zeros((n, 0))
    pca_converged, pca_mvps = True, 0
    if a.k > 0:
        r = svdl(op, GklOptions(k=int(a.k), tol=float(a.tol), max_mvps=int(a.max_mvps),
                                seed=int(a.seed)))
        Z = r.V
        pca_converged, pca_mvps = bool(r.stats.converged), int(r.stats.mvps)
    if a.design:
        X = genio.read_csv_matrix(a.design)
        if X.shape[0] != n:
            raise FormatError(f"{a.design}: design rows do not match samples")
        try:
            if Z.shape[1] > 0:
                fit = R.pc_adjusted_fit(X, Z, y, a.unbiased)
                entry = {"beta": [float(v) for v in fit.beta_hat],
                         "gamma": [float(v) for v in fit.gamma_hat],
                         "sigma2": fit.joint.sigma2_hat}
            else:
                fit = R.ols_fit(X, y, a.unbiased)
                entry = {"beta": [float(v) for v in fit.beta_hat], "sigma2": fit.sigma2_hat}
            entry["se"] = [float(np.sqrt(fit.cov_beta[i, i])) for i in range(fit.beta_hat.size)]
        except R.RankDeficiencyError as e:
            entry = {"error": str(e), "column": e.column}
        result = {"mode": "design", "k": a.k, "pca_converged": pca_converged,
                  "pca_mvps": pca_mvps, "fit": entry}
    else:
        if isinstance(op, DenseOperator):  # .gmx: row statistics on the host matrix
            M = op.apply_block(np.eye(n))
            scan = R.marker_scan(op, y, Z, a.unbiased, sumsq=(M * M).sum(axis=1),
                                 constant=M.max(axis=1) == M.min(axis=1))
        else:
            scan = R.marker_scan(op, y, Z, a.unbiased)
        result = {"mode": "per-marker", "k": a.k, "pca_converged": pca_converged,
                  "pca_mvps": pca_mvps, "markers": R.scan_entries(scan)}
    os.makedirs(a.out, exist_ok=True)
    _write_json(os.path.join(a.out, "regression.json"), result)
    config = {"input": a.input, "pheno": a.pheno, "design": a.design, "k": a.k, "tol": a.tol,
              "max_mvps": a.max_mvps, "standardize": a.standardize, "unbiased": a.unbiased}
    _write_json(os.path.join(a.out, "manifest.json"),
                {"command": "regress", "config": config, "seed": a.seed, "versions": _versions()})
    if not pca_converged:
        sys.stderr.write("gkpca regress: PCA step not converged; results use the partial basis\n")
        return EXIT_UNCONVERGED
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="gkpca", description="Truncated SVD / PCA of genotype matrices on B200")
    p.add_argument("--threads", type=int, default=0,
                   help="accepted for compatibility (host threads are not used on this path)")
    sub = p.add_subparsers(dest="command", parser_class=_Parser)
    c = sub.add_parser("pca", help="Truncated SVD of a genotype/dense matrix")
    c.add_argument("input", help="Input matrix (.gmx or .bed)")
    c.add_argument("--algo", default="gkl", choices=["gkl", "subspace"])
    c.add_argument("-k", "--k", type=int, default=10)
    c.add_argument("--tol", type=float, default=1e-8)
    c.add_argument("--max-mvps", dest="max_mvps", type=int, default=1000000)
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--standardize", default="none", choices=["none", "unit", "binomial", "hwe"])
    c.add_argument("--out", default=".")
    c.add_argument("--reorth", default="partial", choices=["partial", "full"])
    c.add_argument("--omega", type=float, default=1e-8)
    c.add_argument("--restart", default="none", choices=["none", "thick"])
    c.add_argument("--max-subspace", dest="max_subspace", type=int, default=0)
    c.add_argument("--keep", type=int, default=0)
    c.add_argument("--variant", default="qr", choices=["qr", "normalize"])
    c.add_argument("--max-iters", dest="max_iters", type=int, default=1000)
    b = sub.add_parser("bench", help="Compare solvers on one operator with shared mvp counting")
    b.add_argument("input", help="Input matrix (.gmx or .bed)")
    b.add_argument("--algos", default="gkl-pro-nr,gkl-fro-nr,gkl-fro-tr,subspace-qr")
    b.add_argument("-k", "--k", type=int, default=10)
    b.add_argument("--tol", type=float, default=1e-8)
    b.add_argument("--max-mvps", dest="max_mvps", type=int, default=1000000)
    b.add_argument("--max-iters", dest="max_iters", type=int, default=1000)
    b.add_argument("--oracle-cap", dest="oracle_cap", type=int, default=2000)
    b.add_argument("--seed", type=int, required=True)
    b.add_argument("--standardize", default="none", choices=["none", "unit", "binomial", "hwe"])
    b.add_argument("--out", default=".")
    r = sub.add_parser("regress", help="Per-marker regression with PC adjustment")
    r.add_argument("input", help="Genotype matrix (.gmx or .bed)")
    r.add_argument("--pheno", required=True, help="Phenotype CSV (one column, one row per sample)")
    r.add_argument("--design", default="", help="Joint design CSV instead of the per-marker scan")
    r.add_argument("-k", "--k", type=int, default=0)
    r.add_argument("--tol", type=float, default=1e-8)
    r.add_argument("--max-mvps", dest="max_mvps", type=int, default=1000000)
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--standardize", default="none", choices=["none", "unit", "binomial", "hwe"])
    r.add_argument("--unbiased", action="store_true")
    r.add_argument("--out", default=".")
    return p


def main(argv: Optional[List[str]] = None) -> int:
    from ._lib import FormatError
    parser = build_parser()
    try:
        a = parser.parse_args(argv)
        if a.command is None:
            raise UsageError("a subcommand is required")
    except UsageError as e:
        sys.stderr.write(f"gkpca: {e}\n")
        return EXIT_USAGE
    try:
        if a.command == "pca":
            return run_pca(a)
        if a.command == "bench":
            return run_bench(a)
        if a.command == "regress":
            return run_regress(a)
    except FormatError as e:
        sys.stderr.write(f"gkpca: {e}\n")
        return EXIT_FORMAT
    except ValueError as e:  # std::invalid_argument
        sys.stderr.write(f"gkpca: {e}\n")
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001 -- std::exception -> 1 (gkpca.cpp:828-831)
        sys.stderr.write(f"gkpca: {e}\n")
        return 1
    return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
