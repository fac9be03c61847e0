"""PLINK fileset ingest: read_bed's checks (genio.cpp:21-30,53-70) through the
C ABI (gkb_bed_check, CPU) and the streamed file -> HBM loader
(gkb_geno_from_bed_file, GPU) against the payload path."""
import os

import numpy as np
import pytest

from conftest import rel_err


def _fileset(tmp_path, p, n, seed=0, missing=0.02, name="x"):
    from paper_1808_03374_b200 import genio
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 3, size=(p, n)).astype(np.uint8)
    d[rng.random((p, n)) < missing] = 3
    payload = genio.encode(d)
    pre = str(tmp_path / name)
    genio.write_bed(payload, p, n, pre + ".bed", pre + ".bim", pre + ".fam")
    return pre, payload


def test_bed_check_ok_and_counts(gkb, tmp_path):
    pre, _ = _fileset(tmp_path, 13, 29)
    assert gkb.bed_check(pre + ".bed", pre + ".bim", pre + ".fam") == (13, 29)
    # count_lines skips empty lines and counts a last line without newline
    with open(pre + ".bim", "a") as f:
        f.write("\n\n")
    with open(pre + ".fam", "rb+") as f:
        f.seek(-1, os.SEEK_END)
        f.truncate()
    assert gkb.bed_check(pre + ".bed", pre + ".bim", pre + ".fam") == (13, 29)


@pytest.mark.parametrize("content,msg", [
    (b"\x6c\x1a\x01", "bad magic"),
    (b"\x6c", "bad magic"),
    (b"\x6c\x1b\x00", "only marker-major mode (0x01) is supported"),
    (b"\x6c\x1b\x01\x00", "payload size mismatch (expected 107 bytes, found 4)"),
])
def test_bed_check_format_errors(gkb, tmp_path, content, msg):
    pre, _ = _fileset(tmp_path, 13, 29)
    with open(pre + ".bed", "wb") as f:
        f.write(content)
    with pytest.raises(gkb.FormatError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        gkb.bed_check(pre + ".bed", pre + ".bim", pre + ".fam")


def test_bed_check_missing_files(gkb, tmp_path):
    pre, _ = _fileset(tmp_path, 4, 4)
    for bad in ("bed", "bim", "fam"):
        paths = {k: pre + "." + k for k in ("bed", "bim", "fam")}
        paths[bad] = pre + ".nope"
        with pytest.raises(gkb.FormatError, match="cannot open"):
            gkb.bed_check(paths["bed"], paths["bim"], paths["fam"])


def test_bed_check_matches_python_reader(gkb, tmp_path):
    from paper_1808_03374_b200 import genio
    pre, payload = _fileset(tmp_path, 31, 57)
    pay2, p, n = genio.read_bed(pre + ".bed", pre + ".bim", pre + ".fam")
    assert (p, n) == gkb.bed_check(pre + ".bed", pre + ".bim", pre + ".fam")
    assert np.array_equal(pay2, payload)


@pytest.mark.gpu
@pytest.mark.parametrize("p,n,stage_mb,nshards", [(257, 1000, None, 1), (1031, 4099, 1, 1),
                                                  (1031, 4099, 1, 3), (5, 17, None, 2)])
def test_from_bed_file_equals_payload(gkb, tmp_path, monkeypatch, p, n, stage_mb, nshards):
    pre, payload = _fileset(tmp_path, p, n, seed=p + n)
    if stage_mb:
        monkeypatch.setenv("GKB_STAGE_MB", str(stage_mb))  # several double-buffered blocks
    ctx = gkb.Context([0] * nshards) if nshards > 1 else None
    a = gkb.GenotypeOperator.from_bed_file(pre, ctx=ctx)
    b = gkb.GenotypeOperator.from_bed_payload(payload, p, n)
    assert np.array_equal(a.read_bed(), payload)
    assert np.array_equal(a.counts(), b.counts())
    x = np.random.default_rng(3).standard_normal(n)
    ya, yb = a.apply(x), b.apply(x)
    assert rel_err(ya, yb) <= 1e-14
    za, zb = a.apply_adjoint(ya), b.apply_adjoint(yb)
    assert rel_err(za, zb) <= 1e-14


@pytest.mark.gpu
def test_from_bed_file_format_error(gkb, tmp_path):
    pre, _ = _fileset(tmp_path, 8, 9)
    with open(pre + ".bed", "r+b") as f:
        f.write(b"\x00")
    with pytest.raises(gkb.FormatError, match="bad magic"):
        gkb.GenotypeOperator.from_bed_file(pre)
