"""PLINK .bed ingest / egress on the host (genio.cpp:53-122 semantics).

Only the file framing lives here: the payload bytes are handed unchanged to
the device (GenotypeOperator.from_bed_payload), which re-lays and decodes
them in HBM; nothing is densified (load_matrix, gkpca.cpp:89-101, is the
step this replaces).
"""
from __future__ import annotations

import os
from typing import Tuple

import numpy as np

from ._lib import FormatError

MAGIC = bytes([0x6C, 0x1B, 0x01])
CODE_TO_DOSAGE = np.array([2, 3, 1, 0], dtype=np.uint8)   # genio.cpp:33 (3 = missing)
DOSAGE_TO_CODE = np.array([3, 2, 0, 1], dtype=np.uint8)
MISSING = 3


def _count_lines(path: str) -> int:  # genio.cpp:21-30
    try:
        with open(path, "r") as f:
            return sum(1 for line in f if line.rstrip("\n") != "")
    except OSError as e:
        raise FormatError(f"cannot open {path}") from e


def read_bed(bed: str, bim: str, fam: str) -> Tuple[np.ndarray, int, int]:
    """Returns (payload, p, n): the marker-major records after the header,
    checked as read_bed does (genio.cpp:53-70)."""
    p = _count_lines(bim)
    n = _count_lines(fam)
    try:
        raw = np.fromfile(bed, dtype=np.uint8)
    except OSError as e:
        raise FormatError(f"cannot open {bed}") from e
    if raw.size < 3 or raw[0] != 0x6C or raw[1] != 0x1B:
        raise FormatError(f"{bed}: bad magic")
    if raw[2] != 0x01:
        raise FormatError(f"{bed}: only marker-major mode (0x01) is supported")
    stride = (n + 3) // 4
    expected = p * stride + 3
    if raw.size != expected:
        raise FormatError(f"{bed}: payload size mismatch (expected {expected} bytes, "
                          f"found {raw.size})")
    return raw[3:], p, n


def write_bed(payload: np.ndarray, p: int, n: int, bed: str, bim: str, fam: str) -> None:
    """Writes header + payload and placeholder .bim/.fam (genio.cpp:85-122)."""
    payload = np.asarray(payload, dtype=np.uint8)
    if payload.size != p * ((n + 3) // 4):
        raise ValueError("write_bed: payload size does not match p x ceil(n/4)")
    with open(bed, "wb") as f:
        f.write(MAGIC)
        f.write(payload.tobytes())
    with open(bim, "w") as f:
        for i in range(p):
            f.write(f"1\tsnp{i + 1}\t0\t{i + 1}\tA\tB\n")
    with open(fam, "w") as f:
        for s in range(n):
            f.write(f"fam{s + 1}\tind{s + 1}\t0\t0\t0\t-9\n")


def decode(payload: np.ndarray, p: int, n: int) -> np.ndarray:
    """Host decode to a p x n dosage matrix (3 = missing); test/debug helper."""
    stride = (n + 3) // 4
    b = np.asarray(payload, dtype=np.uint8).reshape(p, stride)
    codes = np.stack([(b >> (2 * k)) & 3 for k in range(4)], axis=-1).reshape(p, 4 * stride)
    return CODE_TO_DOSAGE[codes[:, :n]]


def encode(dosages: np.ndarray) -> np.ndarray:
    """p x n dosages (3 = missing) -> payload with 00 pads (genio.cpp:100)."""
    d = np.asarray(dosages, dtype=np.uint8)
    p, n = d.shape
    stride = (n + 3) // 4
    codes = np.zeros((p, 4 * stride), dtype=np.uint8)
    codes[:, :n] = DOSAGE_TO_CODE[d]
    codes = codes.reshape(p, stride, 4)
    out = codes[..., 0] | (codes[..., 1] << 2) | (codes[..., 2] << 4) | (codes[..., 3] << 6)
    return out.astype(np.uint8).reshape(-1)


def bed_paths(prefix: str):
    base = os.path.splitext(prefix)[0] if prefix.endswith(".bed") else prefix
    return base + ".bed", base + ".bim", base + ".fam"


# ---------------------------------------------------------------- GMX1 / CSV
GMX_MAGIC = b"GMX1"


def read_dense(path: str) -> np.ndarray:
    """GMX1 dense matrix (genio.cpp:187-201): 'GMX1', u32 rows, u32 cols, u32
    flags, column-major float64; FormatError on bad magic / size."""
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise FormatError(f"cannot open {path}") from e
    if len(raw) < 16 or raw[:4] != GMX_MAGIC:
        raise FormatError(f"{path}: bad magic")
    m, n = np.frombuffer(raw, dtype="<u4", count=2, offset=4)
    expected = 16 + int(m) * int(n) * 8
    if len(raw) != expected:
        raise FormatError(f"{path}: payload size mismatch (expected {expected} bytes, "
                          f"found {len(raw)})")
    return np.frombuffer(raw, dtype="<f8", offset=16).reshape((int(n), int(m))).T.copy()


def write_dense(path: str, M: np.ndarray, flags: int = 0) -> None:
    """GMX1 writer (genio.cpp:203-217): column-major float64 payload."""
    M = np.asarray(M, dtype=np.float64)
    if M.ndim == 1:
        M = M[:, None]
    try:
        f = open(path, "wb")
    except OSError as e:
        raise FormatError(f"cannot open {path} for writing") from e
    with f:
        f.write(GMX_MAGIC)
        f.write(np.array([M.shape[0], M.shape[1], flags], dtype="<u4").tobytes())
        f.write(np.asfortranarray(M).astype("<f8").tobytes(order="F"))


def write_csv_matrix(path: str, M: np.ndarray) -> None:
    """CSV writer (genio.cpp:261-275): header c1..cN, '%.17g' cells."""
    M = np.asarray(M, dtype=np.float64)
    if M.ndim == 1:
        M = M[:, None]
    try:
        f = open(path, "w")
    except OSError as e:
        raise FormatError(f"cannot open {path} for writing") from e
    with f:
        f.write(",".join(f"c{j + 1}" for j in range(M.shape[1])) + "\n")
        for i in range(M.shape[0]):
            f.write(",".join("%.17g" % v for v in M[i]) + "\n")


def impute_mean(dosages: np.ndarray, return_all_missing: bool = False):
    """impute_mean (genio.cpp:124-148): markers x samples dosages (3 = missing)
    -> float64 with each missing entry replaced by its row's observed mean (0
    for an all-missing row); optionally the all-missing row flags."""
    d = np.asarray(dosages)
    miss = d == 3
    obs = (~miss).sum(axis=1)
    sums = np.where(miss, 0, d).sum(axis=1, dtype=np.float64)
    mean = np.where(obs > 0, sums / np.maximum(obs, 1), 0.0)
    out = np.where(miss, mean[:, None], d.astype(np.float64))
    return (out, obs == 0) if return_all_missing else out


def standardize_dense(X: np.ndarray, scheme: str) -> np.ndarray:
    """standardize (genio.cpp:150-185) on a dense matrix: row mean, population
    variance over all n columns, zero-variance rows -> 0; unit: s = sqrt(var);
    binomial: s = sqrt(q(1-q)), q = clamp(mean/2, 1/(2n+2))."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[1]
    if n == 0:
        raise ValueError("standardize: no samples")
    out = np.zeros_like(X)
    nd = float(n)
    for i in range(X.shape[0]):
        row = X[i]
        mean = row.sum() / nd
        var = ((row - mean) ** 2).sum() / nd
        if var == 0.0:
            continue
        if scheme == "unit":
            s = np.sqrt(var)
        else:
            cl = 1.0 / (2.0 * nd + 2.0)
            q = min(max(mean / 2.0, cl), 1.0 - cl)
            s = np.sqrt(q * (1.0 - q))
        out[i] = (row - mean) / s
    return out


def read_csv_matrix(path: str) -> np.ndarray:
    """read_csv_matrix (genio.cpp:219-259): comma-separated numbers, an optional
    non-numeric header row; FormatError on a non-numeric cell elsewhere, ragged
    rows or no data rows."""
    try:
        f = open(path)
    except OSError as e:
        raise FormatError(f"cannot open {path}") from e
    rows, first = [], True
    with f:
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            row, numeric = [], True
            for cell in line.split(","):
                c = cell.rstrip("\r").rstrip(" ")
                try:
                    row.append(float(c))
                except ValueError:
                    numeric = False
                    break
            if not numeric:
                if first:
                    first = False
                    continue
                raise FormatError(f"{path}: non-numeric cell outside header")
            first = False
            if rows and len(row) != len(rows[0]):
                raise FormatError(f"{path}: ragged rows")
            rows.append(row)
    if not rows:
        raise FormatError(f"{path}: no data rows")
    return np.array(rows, dtype=np.float64)
