"""BASELINE.json workloads: seeded Balding-Nichols genotype specs and the
GklOptions of each config, as plain numpy / dicts.

This module imports nothing from the library (no libgkb.so), so the CPU
reference arm of bench.py and the oracle-side tests can build exactly the
same workload by loading this file on its own. `synth.py` re-exports it for
the product side.

The reference's synth module implements only the paper's Algorithm 1
(proj/src/synth.cpp:24-50); BASELINE's data model is new.
Per-marker subpopulation frequencies (Beta / Dirichlet draws, O(K*p)) are
drawn here with numpy's PCG64; the genotypes themselves (O(n*p)) are drawn
by counter-based hashes keyed by (seed, marker, sample), on the device
(csrc/synth_kernels.cu) or on the CPU by the oracle, bit-identically.

Model: f_j ~ U(0.05, 0.95); p_kj ~ Beta(f(1-F_k)/F_k,
(1-f)(1-F_k)/F_k); g_ij ~ Binomial(2, p_{k(i)j}); equal-size contiguous
subpopulations; missing entries uniform at random (.bed code 01); related
pairs copy the first member's dosage with probability 1/2 per marker;
admixture: q_i ~ Dirichlet(0.5 * 1_K), p_ij = sum_k q_ik p_kj.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

@dataclass
class SynthSpec:
    p: int
    n: int
    seed: int
    freq: np.ndarray                 # npop x p
    pop: Optional[np.ndarray] = None   # n int32
    admix: Optional[np.ndarray] = None  # n x npop
    missing_rate: float = 0.0
    copy_from: Optional[np.ndarray] = None  # n int32 (-1 none)
    copy_prob: float = 0.5
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def npop(self) -> int:
        return int(self.freq.shape[0])

    def to_c(self):
        keep = []

        def ptr(a, ctype):
            if a is None:
                return C.POINTER(ctype)()
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(ctype))

        freq = np.ascontiguousarray(self.freq, dtype=np.float64)
        pop = None if self.pop is None else np.ascontiguousarray(self.pop, dtype=np.int32)
        admix = None if self.admix is None else np.ascontiguousarray(self.admix, dtype=np.float64)
        cf = None if self.copy_from is None else np.ascontiguousarray(self.copy_from, dtype=np.int32)
        from . import _lib  # product-side only (the spec itself is pure numpy)
        s = _lib.gkb_synth_spec()
        s.p, s.n, s.seed, s.npop = self.p, self.n, int(self.seed), self.npop
        s.freq = ptr(freq, C.c_double)
        s.pop = ptr(pop, C.c_int32)
        s.admix = ptr(admix, C.c_double)
        s.missing_rate = float(self.missing_rate)
        s.copy_from = ptr(cf, C.c_int32)
        s.copy_prob = float(self.copy_prob)
        return s, keep

    def sub_block(self, p: int, n: int) -> "SynthSpec":
        """The seeded p x n leading sub-block (identical draws: counter-based)."""
        sb = SynthSpec(p=p, n=n, seed=self.seed, freq=np.ascontiguousarray(self.freq[:, :p]),
                       pop=None if self.pop is None else self.pop[:n].copy(),
                       admix=None if self.admix is None else self.admix[:n].copy(),
                       missing_rate=self.missing_rate,
                       copy_from=None if self.copy_from is None else
                       np.where(self.copy_from[:n] < n, self.copy_from[:n], -1).astype(np.int32),
                       copy_prob=self.copy_prob, name=self.name + f"-sub{p}x{n}")
        return sb


def balding_nichols(n: int, p: int, npop: int, fst, seed: int, missing_rate: float = 0.0,
                    related_pairs: int = 0, admixture_alpha: Optional[float] = None,
                    name: str = "") -> SynthSpec:
    rng = np.random.Generator(np.random.PCG64(seed))
    f = rng.uniform(0.05, 0.95, size=p)
    F = np.broadcast_to(np.asarray(fst, dtype=np.float64), (npop,)).copy()
    freq = np.empty((npop, p))
    for k in range(npop):
        a = f * (1.0 - F[k]) / F[k]
        b = (1.0 - f) * (1.0 - F[k]) / F[k]
        freq[k] = rng.beta(a, b)
    pop = admix = None
    if admixture_alpha is None:
        pop = (np.arange(n, dtype=np.int64) * npop // n).astype(np.int32)
    else:
        admix = rng.dirichlet(np.full(npop, admixture_alpha), size=n)
    copy_from = None
    if related_pairs:
        perm = rng.permutation(n)[: 2 * related_pairs]
        copy_from = np.full(n, -1, dtype=np.int32)
        copy_from[perm[1::2]] = perm[0::2]
    return SynthSpec(p=p, n=n, seed=seed, freq=freq, pop=pop, admix=admix,
                     missing_rate=missing_rate, copy_from=copy_from, copy_prob=0.5, name=name,
                     meta=dict(npop=npop, fst=F.tolist(), related_pairs=related_pairs,
                               admixture_alpha=admixture_alpha))


def config_spec(cfg: int, scale: float = 1.0) -> SynthSpec:
    """BASELINE.json configs[cfg-1] (cfg 1..5); `scale` shrinks n and p for
    parity tests at sizes the CPU oracle finishes in seconds."""
    def sz(v):
        return max(64, int(round(v * scale)))
    if cfg == 1:
        return balding_nichols(sz(2000), sz(20000), 3, 0.01, seed=0, name="C1")
    if cfg == 2:
        return balding_nichols(sz(10000), sz(100000), 5, 0.01, seed=2, missing_rate=0.01,
                               related_pairs=max(1, int(round(50 * min(1.0, scale * 4)))),
                               name="C2")
    if cfg == 3:
        rng = np.random.Generator(np.random.PCG64(1003))
        fst = rng.uniform(0.005, 0.02, size=10)
        return balding_nichols(sz(50000), sz(500000), 10, fst, seed=3, missing_rate=0.005,
                               name="C3")
    if cfg == 4:
        return balding_nichols(sz(500000), sz(100000), 4, 0.01, seed=4, missing_rate=0.01,
                               admixture_alpha=0.5, name="C4")
    if cfg == 5:
        return balding_nichols(sz(1000000), sz(1000000), 8, 0.01, seed=5, missing_rate=0.01,
                               name="C5")
    raise ValueError(f"unknown config {cfg}")


# GklOptions per config as plain fields; reorth 0 = kFull,
# 1 = kPartial; restart 0 = kNone, 1 = kThick. BASELINE gives no restart mode
# for "Krylov dim D": thick restart with keep = max(k, D/2), the CLI default at
# gkpca.cpp:204-209, is the recorded interpretation.
CONFIG_OPTIONS = {
    1: dict(k=10, tol=1e-10, reorth=0, omega=1e-8, restart=1, max_subspace=30, keep=15, seed=0),
    2: dict(k=20, tol=1e-10, reorth=1, omega=1e-8, restart=1, max_subspace=50, keep=25, seed=2),
    3: dict(k=10, tol=1e-10, reorth=1, omega=1e-8, restart=1, max_subspace=40, keep=20, seed=3),
    4: dict(k=20, tol=1e-10, reorth=0, omega=1e-8, restart=1, max_subspace=60, keep=30, seed=4),
    5: dict(k=10, tol=1e-10, reorth=1, omega=1e-8, restart=1, max_subspace=40, keep=20, seed=5),
}

CONFIG_TEXT = {
    1: "config 1: n=2000 x p=20000, 3 subpops, F=0.01, no missing",
    2: "config 2: n=10000 x p=100000, 5 subpops, F=0.01, 1% missing, 50 related pairs",
    3: "config 3: n=50000 x p=500000, 10 subpops, F~U(0.005,0.02), 0.5% missing",
    4: "config 4: n=500000 x p=100000, Dirichlet(0.5) admixture of 4 subpops (F=0.01), 1% missing",
    5: "config 5: n=1000000 x p=1000000, 8 subpops, F=0.01, 1% missing",
}

OPTIONS_TEXT = {
    1: "full reorth, thick restart 30/15, tol 1e-10, seed 0",
    2: "partial reorth w=1e-8 (complete omega recurrence, non-reference), thick restart 50/25, "
       "tol 1e-10, seed 2",
    3: "partial reorth w=1e-8 (complete omega recurrence, non-reference), thick restart 40/20, "
       "tol 1e-10, seed 3",
    4: "full reorth, thick restart 60/30, tol 1e-10, seed 4",
    5: "partial reorth w=1e-8 (complete omega recurrence, non-reference), thick restart 40/20, "
       "tol 1e-10, seed 5",
}
