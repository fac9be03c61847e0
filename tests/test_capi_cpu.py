"""C ABI checks that need no GPU: the library loads, exports every entry
point include/gkb.h declares, and its host-only logic (row partition, host
Jacobi svd_small, marker scaling, Rng, option validation) matches the
oracle / LAPACK."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1808_03374_b200 as gkb
from paper_1808_03374_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "gkb.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(gkb_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = declared_symbols()
    assert len(names) >= 35
    lib = C.CDLL(_lib.LIB_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


@pytest.mark.parametrize("m,parts", [(0, 1), (1, 1), (5, 2), (17, 3), (100000, 8), (7, 8)])
def test_partition_rows(m, parts):
    st = gkb.partition_rows(m, parts)
    assert st[0] == 0 and st[-1] == m and np.all(np.diff(st) >= 0)
    assert all(s % 4 == 0 for s in st[1:-1] if s < m)
    if m >= 4 * parts:
        sizes = np.diff(st)
        assert sizes.max() - sizes.min() <= 4


@pytest.mark.parametrize("shape", [(1, 1), (3, 3), (10, 10), (20, 7), (7, 20), (40, 41), (64, 64)])
def test_host_svd_small_vs_lapack(shape):
    M = O.gaussian_matrix(shape[0], shape[1], 17 + shape[0])
    U, s, V = gkb.svd_small(M)
    k = min(shape)
    assert np.allclose(s, np.linalg.svd(M, compute_uv=False), rtol=0, atol=1e-12 * s[0])
    assert np.abs(U.T @ U - np.eye(k)).max() <= 1e-12
    assert np.abs(V.T @ V - np.eye(k)).max() <= 1e-12
    assert np.abs(U @ np.diag(s) @ V.T - M).max() <= 1e-12 * s[0]


def test_host_svd_rank_deficient_completion():
    # compress_exhausted's augmented [B | coupling] can be rank deficient:
    # both factors must stay orthonormal (null directions completed)
    B = np.diag([3.0, 2.0, 0.0, 0.0])
    aug = np.hstack([B, np.zeros((4, 1))])
    U, s, V = gkb.svd_small(aug)
    assert np.allclose(s, [3, 2, 0, 0])
    assert np.abs(U.T @ U - np.eye(4)).max() <= 1e-14
    assert np.abs(V.T @ V - np.eye(4)).max() <= 1e-14


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_marker_scaling_bit_exact_vs_oracle(scheme):
    r = np.random.default_rng(scheme)
    n = 997
    counts = []
    for _ in range(500):
        k = r.integers(0, 4)
        parts = r.multinomial(n, r.dirichlet(np.ones(4)))
        if k == 0:
            parts = np.array([n, 0, 0, 0])
        elif k == 1:
            parts = np.array([0, 0, 0, n])
        counts.append(parts)
    counts = np.array(counts, dtype=np.int64)
    mu, inv_s = gkb.marker_scaling(counts, n, gkb.ScalingScheme(scheme))
    mu_o, is_o = O.marker_scaling(counts, n, scheme)
    assert np.array_equal(mu, mu_o) and np.array_equal(inv_s, is_o)


def test_rng_matches_oracle_bitwise():
    for seed in (0, 1, 99, 2**63 + 5):
        assert np.array_equal(gkb.rng_uniform_symmetric(seed, 1000), O.rng_fill_symmetric(seed, 1000))


def test_option_validation_messages():
    cases = [(dict(k=9), "k must lie"), (dict(k=0), "k must lie"), (dict(k=2, tol=0.0), "tol"),
             (dict(k=2, max_mvps=1), "max_mvps"), (dict(k=2, omega=0.0), "omega"),
             (dict(k=2, restart=gkb.RestartMode.kThick, max_subspace=6, keep=6), "below"),
             (dict(k=2, restart=gkb.RestartMode.kThick, max_subspace=6, keep=1), "at least k"),
             (dict(k=2, restart=gkb.RestartMode.kThick, max_subspace=100, keep=4), "exceed")]
    for kw, msg in cases:
        with pytest.raises(ValueError, match=msg):
            gkb.GklOptions(**kw).validate(10, 8)
        with pytest.raises(ValueError, match=msg):
            O.validate(O.Options.from_gkl(gkb.GklOptions(**kw)), 10, 8)
    gkb.GklOptions(k=2).validate(10, 8)


def test_no_gpu_fails_loudly():
    """Without a device the CUDA path raises; nothing falls back to the CPU."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(gkb.GkbError):
        gkb.Context((0,))


def test_genio_roundtrip(tmp_path):
    from paper_1808_03374_b200 import genio
    r = np.random.default_rng(99)
    d = r.integers(0, 4, size=(7, 13)).astype(np.uint8)
    pay = genio.encode(d)
    assert np.array_equal(pay, O.bed_encode(d))
    bed, bim, fam = genio.bed_paths(str(tmp_path / "x"))
    genio.write_bed(pay, 7, 13, bed, bim, fam)
    back, p, n = genio.read_bed(bed, bim, fam)
    assert (p, n) == (7, 13) and np.array_equal(back, pay)
    assert np.array_equal(genio.decode(back, p, n), d)
    with open(bed, "r+b") as f:
        f.write(b"\x00")
    with pytest.raises(gkb.FormatError):
        genio.read_bed(bed, bim, fam)


def test_layout_planner():
    """gkb_geno_plan (host-only): config 5 at 2 GPUs (500,000 SNPs x 1,000,000
    samples per GPU, 1% missing) does not fit two 125 GB layouts in a B200's
    HBM and plans one (~154 GB); config 4 on one GPU keeps both."""
    import paper_1808_03374_b200 as gkb
    hbm = 178 << 30
    layouts, dual, single = gkb.geno_plan(500_000, 1_000_000, 0.01, hbm)
    assert layouts == 1 and dual > hbm and single < hbm
    assert single >= 125_000_000_000
    layouts, dual, single = gkb.geno_plan(100_000, 500_000, 0.01, hbm)
    assert layouts == 2 and dual < hbm
    assert gkb.geno_plan(250_000, 1_000_000, 0.01, hbm)[0] == 2   # config 5 at 4 GPUs
