"""Generates tests/golden/c5_sub_100k.npz: the CPU oracle's svdl on the seeded
100,000 x 100,000 leading sub-block of BASELINE config 5 (SURVEY.md 8d:
"CPU oracle run on a 100,000 x 100,000 seeded sub-block for tolerance
checks"), with config 5's GklOptions (k=10, partial reorth w=1e-8, thick
restart 40/20, tol 1e-10, seed 5) and hwe standardization.

Test infrastructure: runs the oracle restatement (oracle/, OpenMP) on the
CPU; about 10-20 minutes on 8 cores. Stored: the top-k singular values and
error estimates (float64), the solver's counters, and the QR-orthonormalized
U (SNP side) and V (sample side) Ritz bases as float32 (the rounding moves
the subspaces by ~1e-8 radians, far below the 1e-6 parity bound), plus the
sha256 of the sub-block's .bed payload so a changed generator is detected.

usage: python tests/golden/make_c5_subblock.py [nthreads]
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (workloads loader: pure numpy, no libgkb)
import oracle  # noqa: E402

SUB = 100_000


def main():
    nthreads = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    W = bench.load_workloads()
    spec = W.config_spec(5).sub_block(SUB, SUB)
    t0 = time.time()
    payload = oracle.synth_bed(spec)
    digest = hashlib.sha256(payload.tobytes()).hexdigest()
    counts = oracle.marker_counts(payload, spec.p, spec.n)
    mu, inv_s = oracle.marker_scaling(counts, spec.n, 2)
    g = oracle.GenoOracle(payload, spec.p, spec.n, mu, inv_s, nthreads=nthreads)
    opts = oracle.Options(**W.CONFIG_OPTIONS[5])
    print(f"generated in {time.time() - t0:.1f}s; solving ...", flush=True)
    t0 = time.time()
    r = oracle.svdl(g, opts)
    el = time.time() - t0
    qu = np.linalg.qr(r.U)[0].astype(np.float32)
    qv = np.linalg.qr(r.V)[0].astype(np.float32)
    out = os.path.join(HERE, "c5_sub_100k.npz")
    np.savez(out, singvals=r.singvals, err=r.err, U=qu, V=qv,
             mvps=r.mvps, steps=r.steps, restarts=r.restarts,
             converged=r.all_converged, payload_sha256=digest,
             omega_recurrence=opts.omega_recurrence, seconds=el, nthreads=nthreads)
    print(f"svdl {el:.1f}s mvps={r.mvps} restarts={r.restarts} conv={r.all_converged}")
    print("singvals", r.singvals)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
