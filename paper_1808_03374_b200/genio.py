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
