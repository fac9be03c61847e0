"""The library's multi-process (SPMD) path, run as 2 processes on ONE GPU.

NCCL cannot place two ranks on one device, so each rank's context is made
with gkb_init_host_comm: the library's collectives -- the adjoint's length-n
allreduce (linop.hpp:55-58 under SNP sharding), the U-basis Gram-Schmidt
partials (orth.hpp:19-44), the MGS second-pass dots, the gathers of U / y --
run through the same SPMD branches as with NCCL, with the sum done by
torch.distributed over gloo in a CUDA host function (stream-ordered D2H ->
host sum -> H2D; no kernel waits on the other process). Each rank owns the
SNP shard of gkb_partition_rows. Results must equal the single-process
solve: the products bit-for-bit on the shard-local side and to fp64
reassociation after the sums; svdl to 1e-9 per sigma with principal angles
< 1e-6 and the same counters.
"""
import os
import socket

import numpy as np
import pytest

from conftest import principal_angles, rel_err, sigma_rel_err

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, host_step, env=None):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if host_step:
        os.environ["GKB_HOST_STEP"] = "1"
    os.environ.update(env or {})
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        import paper_1808_03374_b200 as gkb
        from paper_1808_03374_b200 import subspace as Sb
        from paper_1808_03374_b200 import synth

        def allreduce(a):
            dist.all_reduce(torch.from_numpy(a))

        ctx = gkb.Context(host_comm=(0, world, rank, allreduce))
        for cfg, scale in [(2, 0.05), (3, 0.01)]:
            spec = synth.config_spec(cfg, scale=scale)
            opts = synth.config_options(cfg)
            op = gkb.GenotypeOperator.from_synth(spec, ctx=ctx, scheme=gkb.ScalingScheme.kHwe)
            rng = np.random.default_rng(cfg)
            x = rng.standard_normal(spec.n)
            y = op.apply(x)
            z = op.apply_adjoint(y)
            res = gkb.svdl(op, opts)
            sres = Sb.subspace_iterate(op, 4, Sb.SubspaceVariant.kQr, 1e-8, 12, 0)
            out[cfg] = dict(y=y.copy(), z=z.copy(), s=res.singvals.copy(), U=np.array(res.U),
                            V=np.array(res.V), mvps=res.stats.mvps, restarts=res.stats.restarts,
                            steps=res.stats.steps, reorth=res.stats.reorth_count,
                            conv=res.stats.converged, mu=op.scaling()[0].copy(),
                            sub_s=np.array(sres.state.singvals if hasattr(sres.state, "singvals")
                                           else sres.singvals),
                            sub_mvps=sres.mvps)
            op.close()
        ctx.close()
        if rank == 0:
            q.put(out)
    except BaseException:
        import traceback
        traceback.print_exc()
        if rank == 0:
            q.put(None)
        raise
    finally:
        dist.destroy_process_group()


def _single(gkb, cfg, scale, host_step, monkeypatch, env=None):
    from paper_1808_03374_b200 import subspace as Sb
    from paper_1808_03374_b200 import synth
    if host_step:
        monkeypatch.setenv("GKB_HOST_STEP", "1")
    for key, val in (env or {}).items():
        monkeypatch.setenv(key, val)
    spec = synth.config_spec(cfg, scale=scale)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    rng = np.random.default_rng(cfg)
    x = rng.standard_normal(spec.n)
    y = op.apply(x)
    z = op.apply_adjoint(y)
    res = gkb.svdl(op, synth.config_options(cfg))
    sres = Sb.subspace_iterate(op, 4, Sb.SubspaceVariant.kQr, 1e-8, 12, 0)
    monkeypatch.delenv("GKB_HOST_STEP", raising=False)
    return dict(y=y, z=z, s=res.singvals, U=np.array(res.U), V=np.array(res.V),
                mvps=res.stats.mvps, restarts=res.stats.restarts, steps=res.stats.steps,
                reorth=res.stats.reorth_count, conv=res.stats.converged, mu=op.scaling()[0],
                sub_s=np.array(sres.state.singvals if hasattr(sres.state, "singvals")
                               else sres.singvals), sub_mvps=sres.mvps)


MODES = [(False, {}), (True, {}),
         # single-layout adjoint, dense-missing indicator MMAs, tcgen05 block products
         (False, {"GKB_LAYOUTS": "1", "GKB_MISS_MODE": "ind", "GKB_TC_BLOCK": "1"})]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("host_step,env", MODES, ids=["device-step", "host-step", "modes"])
def test_two_process_spmd_equals_single_process(gkb, monkeypatch, host_step, env):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, host_step, env)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=540)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert got is not None
    for cfg, scale in [(2, 0.05), (3, 0.01)]:
        a, b = got[cfg], _single(gkb, cfg, scale, host_step, monkeypatch, env)
        assert np.array_equal(a["mu"], b["mu"])            # global marker counts -> same scaling
        assert np.array_equal(a["y"], b["y"])              # K1 is shard-local: bitwise
        assert rel_err(a["z"], b["z"]) <= 1e-14            # K2 partials + allreduce
        assert sigma_rel_err(a["s"], b["s"]) <= 1e-9
        assert principal_angles(a["U"], b["U"]) < 1e-6
        assert principal_angles(a["V"], b["V"]) < 1e-6
        assert a["conv"] == b["conv"]
        assert abs(a["restarts"] - b["restarts"]) <= 1
        assert sigma_rel_err(a["sub_s"], b["sub_s"]) <= 1e-9
        assert a["sub_mvps"] == b["sub_mvps"]
    for key in (env or {}):
        monkeypatch.delenv(key, raising=False)


def _nccl_worker(q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["GKB_NCCL_FORCE"] = "1"
    try:
        import paper_1808_03374_b200 as gkb
        from paper_1808_03374_b200 import synth
        uid = gkb.Context.nccl_unique_id()
        ctx = gkb.Context(nccl=(0, uid, 1, 0))
        spec = synth.config_spec(2, scale=0.05)
        op = gkb.GenotypeOperator.from_synth(spec, ctx=ctx, scheme=gkb.ScalingScheme.kHwe)
        x = np.random.default_rng(2).standard_normal(spec.n)
        y = op.apply(x)
        z = op.apply_adjoint(y)
        res = gkb.svdl(op, synth.config_options(2))
        q.put(dict(y=y.copy(), z=z.copy(), s=res.singvals.copy(), U=np.array(res.U),
                   V=np.array(res.V), mvps=res.stats.mvps, mu=op.scaling()[0].copy()))
        op.close()
        ctx.close()
    except BaseException:
        import traceback
        traceback.print_exc()
        q.put(None)
        raise


@pytest.mark.timeout(300)
def test_nccl_one_rank_equals_default_context(gkb):
    """A one-rank NCCL context (gkb_init_nccl) with GKB_NCCL_FORCE=1 sends
    every allreduce of the SPMD branches through ncclAllReduce (an identity
    for one rank): the solve must be bitwise the default context's. This runs
    the NCCL plumbing (comm init, allreduces enqueued on the library's stream)
    on a one-GPU box; sums across ranks are covered by the host-comm tests."""
    import torch.multiprocessing as mp
    from paper_1808_03374_b200 import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_worker, args=(q,))
    pr.start()
    got = q.get(timeout=280)
    pr.join(timeout=60)
    assert got is not None and pr.exitcode == 0
    spec = synth.config_spec(2, scale=0.05)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    x = np.random.default_rng(2).standard_normal(spec.n)
    assert np.array_equal(got["mu"], op.scaling()[0])
    assert np.array_equal(got["y"], op.apply(x))
    assert np.array_equal(got["z"], op.apply_adjoint(got["y"]))
    res = gkb.svdl(op, synth.config_options(2))
    assert np.array_equal(got["s"], res.singvals)
    assert np.array_equal(got["U"], np.array(res.U)) and np.array_equal(got["V"], np.array(res.V))
    assert got["mvps"] == res.stats.mvps
    op.close()
