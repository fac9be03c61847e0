"""World-size-2 CPU test of the multi-GPU decomposition with torch.distributed
(gloo). Each rank owns the SNP shard given by the product's own row
partition (gkb_partition_rows); the shard-local work is evaluated with the
oracle's row-range operators and the cross-rank sums with gloo allreduce --
the same placement libgkb uses with NCCL:
  apply (A^T u, reference X x)        : shard-local, no collective
  apply_adjoint (A v, reference X^T y): allreduce(sum) of n partials
  U-basis Gram-Schmidt dot products   : allreduce(sum) of j+1 partials
The assembled results must equal the unsharded oracle to fp64 reassociation.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_1808_03374_b200 as gkb
        from paper_1808_03374_b200 import synth

        spec = synth.config_spec(2, scale=0.02)
        p, n = spec.p, spec.n
        payload = O.synth_bed(spec)
        mu, inv_s = O.marker_scaling(O.marker_counts(payload, p, n), n, 2)
        g = O.GenoOracle(payload, p, n, mu, inv_s)
        st = gkb.partition_rows(p, world)
        j0, j1 = int(st[rank]), int(st[rank + 1])
        rng = np.random.default_rng(5)
        x = rng.standard_normal(n)
        y = rng.standard_normal(p)
        # apply: local rows only
        y_loc = g.apply_rows(j0, j1, x)
        full = torch.zeros(p, dtype=torch.float64)
        full[j0:j1] = torch.from_numpy(y_loc)
        dist.all_reduce(full)
        # adjoint: partial over local SNPs, allreduce n
        z = torch.from_numpy(g.apply_adjoint_rows(j0, j1, y[j0:j1]).copy())
        dist.all_reduce(z)
        # left-basis CGS coefficients: local Gram partials + norm, allreduce j+1
        U = rng.standard_normal((p, 6))
        w = rng.standard_normal(p)
        part = torch.from_numpy(np.concatenate([U[j0:j1].T @ w[j0:j1], [w[j0:j1] @ w[j0:j1]]]))
        dist.all_reduce(part)
        # timing reduction: max over ranks
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put(dict(y=full.numpy(), y_ref=g.apply(x), z=z.numpy(), z_ref=g.apply_adjoint(y),
                       c=part.numpy(), c_ref=np.concatenate([U.T @ w, [w @ w]]), tmax=t.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world_size_2_sharded_decomposition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert np.array_equal(res["y"], res["y_ref"])          # shard-local rows: bitwise
    assert np.max(np.abs(res["z"] - res["z_ref"])) <= 1e-12 * np.max(np.abs(res["z_ref"]))
    assert np.max(np.abs(res["c"] - res["c_ref"])) <= 1e-12 * np.max(np.abs(res["c_ref"]))
    assert res["tmax"] == 2.0
