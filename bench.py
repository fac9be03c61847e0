#!/usr/bin/env python
"""Benchmark of the B200 GKL hot path (BASELINE.json metric).

Headline metric: packed genotype matvec HBM GB/s (A*v + A^T*u), plus seconds
to the top-k singular triplets. Default workload: BASELINE config 4, the
largest single-GPU config (n = 500,000 individuals x p = 100,000 SNPs,
Dirichlet(0.5) admixture of 4 Balding-Nichols subpopulations, F = 0.01, 1%
missing; 12.5 GB packed), generated on the device by the seeded
counter-based generator (synthetic data of the config's model; BASELINE names
no public dataset). `--config 3` selects config 3 (6.25 GB packed).

A step is one reference apply (A^T u, per-SNP dot, kernel K1) plus one
apply_adjoint (A v, per-sample sum, kernel K2) on device-resident vectors;
`value` = 2 * packed bytes of the whole matrix / step time. Each product is
digitize + main + a fixed-order partial-sum reduce.

  python bench.py [--config 4] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU over NCCL: STRONG scaling -- the
config's SNPs are partitioned across the ranks (each owns ~p/N SNPs), K1 is
shard-local and K2's length-n partial sums are combined with ncclAllReduce;
`time_to_solution` is the sharded svdl.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle restatement in oracle/, the reference itself cannot be built here: no
Eigen / vendor/) with all host threads on a bounded SNP sample of the SAME
config, and never loads libgkb: the workload spec comes from
paper_1808_03374_b200/workloads.py loaded by file path (pure numpy).
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEFAULT_CFG = 4
METRIC = "packed genotype matvec HBM GB/s (A·v+Aᵀ·u); seconds to top-k singular triplets"
# ncu --set full captures of the main kernels per config (tools/ncu_summary.py)
NCU_CAPTURE = {4: "r2d_ncu_full_config4.json", 2: "r1j_ncu_full_config2.json"}


def load_workloads():
    """paper_1808_03374_b200/workloads.py by path: the package (and libgkb)
    is never imported on the reference arm."""
    name = "_gkb_workloads"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(
        name, os.path.join(ROOT, "paper_1808_03374_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([v.strip() for v in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, nm in enumerate(names):
                if len(s) > 4 + k and s[4 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def ncu_traffic(cfg: int, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` capture of this workload (profiles/)."""
    name = NCU_CAPTURE.get(cfg)
    if not name:
        return None
    p = os.path.join(ROOT, "profiles", name)
    try:
        with open(p) as f:
            d = json.load(f)
        m = d[kernel]

        def mb(s):
            v, u = s.split()[:2]
            return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        return (int(mb(m["dram__bytes_read.sum"]) + mb(m["dram__bytes_write.sum"])), name)
    except Exception:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_block(W, cfg, spec, ws):
    """The `config` object; identical on both arms (same workload)."""
    return {"workload": W.CONFIG_TEXT[cfg] + ", hwe standardization (g-2f)/sqrt(2f(1-f))",
            "config_index": cfg, "n": spec.n, "p": spec.p,
            "packed_bytes": spec.p * ((spec.n + 3) // 4),
            "options": W.OPTIONS_TEXT[cfg],
            "l2": "inputs larger than L2 (two multi-GB tile layouts alternate; no flush)",
            "parallelism": f"snp-shard{ws}"}


# ---------------------------------------------------------------- CPU legs
def cpu_port_sample(W, spec, rows: int, nthreads: int, min_seconds: float,
                    max_steps: int = 1000, row0: int = 0):
    """Times the oracle's packed operator (apply + apply_adjoint) on SNPs
    [row0, row0 + rows) of the workload. Returns (GB/s, steps, seconds)."""
    import oracle
    payload = oracle.synth_bed(spec, row0, row0 + rows)
    counts = oracle.marker_counts(payload, rows, spec.n)
    mu, inv_s = oracle.marker_scaling(counts, spec.n, 2)
    g = oracle.GenoOracle(payload, rows, spec.n, mu, inv_s, nthreads=nthreads)
    x = oracle.rng_fill_symmetric(7, spec.n)
    x /= np.linalg.norm(x)
    y = g.apply(x)
    steps, t0 = 0, time.perf_counter()
    while True:
        y = g.apply(x)
        g.apply_adjoint(y)
        steps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or steps >= max_steps:
            break
    bytes_step = 2 * rows * ((spec.n + 3) // 4)
    return bytes_step * steps / el / 1e9, steps, el


def cpu_dense_svdl(W, cfg: int):
    """The reference's literal CPU path on config `cfg` (1 thread, as the
    reference runs): .bed bytes -> dense fp64 impute_mean + standardize
    (load_matrix, gkpca.cpp:89-108; genio.cpp:124-185) -> DenseOperator
    (linop.hpp:43-64) -> svdl (gkl.cpp:416-514), restated in oracle/."""
    import oracle
    spec = W.config_spec(cfg)
    payload = oracle.synth_bed(spec)
    counts = oracle.marker_counts(payload, spec.p, spec.n)
    mu, inv_s = oracle.marker_scaling(counts, spec.n, 2)
    t0 = time.perf_counter()
    X = oracle.dense_standardized(payload, spec.p, spec.n, mu, inv_s)
    t_pre = time.perf_counter() - t0
    opts = oracle.Options(**W.CONFIG_OPTIONS[cfg])
    t0 = time.perf_counter()
    r = oracle.svdl(oracle.DenseOracle(X), opts)
    t = time.perf_counter() - t0
    return {"config": cfg, "seconds": round(t, 3), "preprocess_seconds": round(t_pre, 3),
            "mvps": r.mvps, "steps": r.steps, "restarts": r.restarts,
            "converged": bool(r.all_converged), "cores": 1,
            "sigma_1": float(r.singvals[0]) if r.singvals.size else None,
            "path": "oracle dense (densified fp64 matrix, column-major GEMV) svdl, 1 thread"}


def run_reference(args):
    """CPU reference arm: the oracle restatement of the reference's operator,
    all host threads, on a bounded SNP sample of the same config."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    W = load_workloads()
    cfg = args.config
    spec = W.config_spec(cfg)
    cores = os.cpu_count() or 1
    stride = (spec.n + 3) // 4
    # ~1 GB of packed rows per product: a step is ~1 s of 16-core CPU work
    rows = max(64, min(spec.p, int(1e9 // stride)))
    vals = []
    for _ in range(args.warmup):
        cpu_port_sample(W, spec, min(rows, 256), cores, 0.0, max_steps=1)
    import oracle
    payload = oracle.synth_bed(spec, 0, rows)
    counts = oracle.marker_counts(payload, rows, spec.n)
    mu, inv_s = oracle.marker_scaling(counts, spec.n, 2)
    g = oracle.GenoOracle(payload, rows, spec.n, mu, inv_s, nthreads=cores)
    x = oracle.rng_fill_symmetric(7, spec.n)
    x /= np.linalg.norm(x)
    g.apply_adjoint(g.apply(x))
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        y = g.apply(x)
        g.apply_adjoint(y)
        vals.append(2 * rows * stride / (time.perf_counter() - t0) / 1e9)
    el = time.perf_counter() - t_all
    v = 2 * rows * stride * args.steps / el / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator of the config's BASELINE model)",
        "config": config_block(W, cfg, spec, ws),
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"oracle packed operator apply+apply_adjoint (OpenMP, {cores} "
                                   f"threads) on SNPs [0,{rows}) of config {cfg} "
                                   f"({2 * rows * stride / 1e9:.2f} GB per step); the full "
                                   f"config is {spec.p} SNPs", "step_gbs_median":
                                   round(statistics.median(vals), 4)},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import paper_1808_03374_b200 as gkb
    from paper_1808_03374_b200 import synth

    W = load_workloads()
    cfg = args.config
    ws, rank, local = dist_env()
    dist = None
    host_comm = os.environ.get("GKB_BENCH_HOST_COMM") == "1"
    if ws > 1 and host_comm:
        # test mode for the N > 1 harness on a box with fewer GPUs than ranks:
        # every rank on device 0, the library's sums over gloo through
        # gkb_init_host_comm (timings are not NVLink numbers)
        import torch
        import torch.distributed as tdist
        local = 0
        torch.cuda.set_device(0)
        tdist.init_process_group("gloo")
        sum_group = tdist.new_group(backend="gloo")

        def host_allreduce(a):
            tdist.all_reduce(torch.from_numpy(a), group=sum_group)
        ctx = gkb.Context(host_comm=(0, ws, rank, host_allreduce))
        dist = tdist
    elif ws > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        uid = gkb.Context.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device=f"cuda:{local}")
        tdist.broadcast(t, 0)
        uid = bytes(t.cpu().tolist())
        ctx = gkb.Context(nccl=(local, uid, ws, rank))
        dist = tdist
    else:
        ctx = gkb.Context((0,))

    def barrier():
        ctx.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if not dist:
            return v
        import torch
        tt = torch.tensor([v], dtype=torch.float64,
                          device="cpu" if host_comm else f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # strong scaling: the config's SNPs partitioned across the ranks
    spec = synth.config_spec(cfg)
    t_build = time.perf_counter()
    op = gkb.GenotypeOperator.from_synth(spec, ctx=ctx, scheme=gkb.ScalingScheme.kHwe)
    ctx.synchronize()
    t_build = time.perf_counter() - t_build
    info = op.info()
    packed_local = info["packed_bytes"]
    packed_total = spec.p * ((spec.n + 3) // 4)

    # warm-up steps, then per-kernel timings (device events on the library's
    # stream) and the timed region; nvidia-smi samples clocks across this whole
    # window (the same kernels back to back) so the timed region is covered.
    op.bench(2, args.warmup, flush_l2=False)
    barrier()
    with ClockSampler(local) as clk:
        iters_k = max(args.steps, int(0.4 / max(1e-6, 0.15e-3 * packed_local / 250e6)))
        # K1 and K2 timed in alternating chunks: under the power cap the SM
        # clock drifts down while the GPU heats, so timing one kernel's block
        # after the other's would charge the drift to the second
        nchunk = 4
        per = max(1, iters_k // nchunk)
        t = [[0.0, 0.0], [0.0, 0.0]]
        for _ in range(nchunk):
            for kind in (0, 1):
                ms, main, _ = op.bench(kind, per, flush_l2=False)
                t[kind][0] += ms / nchunk
                t[kind][1] += main / nchunk
        (k1_ms, k1_main), (k2_ms, k2_main) = t
        barrier()
        step_ms, main_ms, launches = op.bench(2, args.steps, flush_l2=False)
        barrier()
    clocks = clk.summary()
    step_ms = max_over_ranks(step_ms)
    value = 2 * packed_total / (step_ms * 1e-3) / 1e9

    # e2e through the public API with host buffers (H2D inputs, D2H results)
    # (page-locked numpy arrays from gkb.pinned_empty, used in place)
    rng = np.random.default_rng(7)
    x = gkb.pinned_empty(spec.n)
    x[:] = rng.standard_normal(spec.n)
    x /= np.linalg.norm(x)
    y = gkb.pinned_empty(spec.p)
    z = gkb.pinned_empty(spec.n)
    for _ in range(args.warmup):
        op.apply(x, out=y)
        op.apply_adjoint(y, out=z)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.apply(x, out=y)
        op.apply_adjoint(y, out=z)
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    e2e = 2 * packed_total / e2e_s / 1e9
    h2d = 8 * (spec.n + spec.p) * ws   # x (n) for apply, y (p) for the adjoint, every rank
    d2h = 8 * (spec.p + spec.n) * ws   # y (p) and z (n) read back

    # .bed file -> HBM ingest on a leading SNP block of the
    # workload written as a PLINK fileset (page-cache-warm file)
    ingest = None
    if rank == 0 and ws == 1 and not args.no_ingest:
        import tempfile
        from paper_1808_03374_b200 import genio
        rows = min(spec.p, max(4096, int(1.0e9 // ((spec.n + 3) // 4))))
        with tempfile.TemporaryDirectory() as td:
            pre = os.path.join(td, "blk")
            genio.write_bed(op.read_bed(0, rows), rows, spec.n, pre + ".bed", pre + ".bim",
                            pre + ".fam")
            op_f = gkb.GenotypeOperator.from_bed_file(pre, ctx=ctx)  # warm the page cache
            op_f.close()
            t0 = time.perf_counter()
            op_f = gkb.GenotypeOperator.from_bed_file(pre, ctx=ctx)
            ctx.synchronize()
            t_in = time.perf_counter() - t0
            op_f.close()
        fbytes = rows * ((spec.n + 3) // 4) + 3
        ingest = {"seconds": round(t_in, 4), "bytes": fbytes, "gbs": round(fbytes / t_in / 1e9, 2),
                  "note": f"page-cache-warm .bed of SNPs [0,{rows}) of the workload -> HBM: "
                          "header/size checks, streamed positional reads + both tile layouts, "
                          "marker counts, missing lists, scaling"}

    # time to top-k triplets (the config's BASELINE options)
    opts = synth.config_options(cfg)
    barrier()
    t0 = time.perf_counter()
    res = gkb.svdl(op, opts)
    tts_first = max_over_ranks(time.perf_counter() - t0)  # includes the solver's buffers
    barrier()
    t0 = time.perf_counter()
    res = gkb.svdl(op, opts)
    tts = max_over_ranks(time.perf_counter() - t0)

    # widened rows on the same operator: subspace iteration
    # (QR variant, device-resident blocks; a bounded 40-iteration sample) and
    # the per-marker PC-adjusted regression scan with the solve's first 10 PCs
    widened = None
    if rank == 0 and ws == 1 and not args.no_widen:
        from paper_1808_03374_b200 import regress as Rg
        from paper_1808_03374_b200 import subspace as Sb
        t0 = time.perf_counter()
        sres = Sb.subspace_iterate(op, 10, Sb.SubspaceVariant.kQr, 1e-8, 40, 0)
        t_sub = time.perf_counter() - t0
        pheno = np.random.default_rng(11).standard_normal(spec.n)
        Zpc = res.V[:, :10]
        Rg.marker_scan(op, pheno, Zpc)  # warm-up (block buffers)
        t0 = time.perf_counter()
        scan = Rg.marker_scan(op, pheno, Zpc)
        t_reg = time.perf_counter() - t0
        widened = {
            "subspace": {"seconds": round(t_sub, 4), "k": 10, "iterations": sres.state.iterations,
                         "mvps": sres.mvps, "converged": bool(sres.converged),
                         "matvec_gbs": round(sres.mvps * packed_local / t_sub / 1e9, 1),
                         "sample": "subspace_iterate kQr, k=10, tol 1e-8, max 40 iterations"},
            "regress": {"seconds": round(t_reg, 4), "markers": int(scan.beta.size),
                        "markers_per_s": round(scan.beta.size / t_reg, 1), "pcs": 10,
                        "sample": "marker_scan: y ~ [1, m_i, Z] for every SNP (12-column block "
                                  "product, two columns per pass, and per-marker algebra on "
                                  "the device)"},
        }

    peak, peak_src = load_peaks()
    b_mvp = packed_local
    k1_gbs = b_mvp / (k1_main * 1e-3) / 1e9
    k2_gbs = b_mvp / (k2_main * 1e-3) / 1e9
    # dominant kernel = the slower of the two main kernels (k_pm_main<1> = K2
    # apply_adjoint, k_pm_main<0> = K1 apply); its average launch duration
    # from CUDA events on the library's stream
    dom = ("K2 apply_adjoint (A·v): k_pm_main<1>", k2_gbs, k2_main, "k_pm_main<1>") \
        if k2_main >= k1_main else ("K1 apply (Aᵀ·u): k_pm_main<0>", k1_gbs, k1_main, "k_pm_main<0>")
    traffic = ncu_traffic(cfg, dom[3]) if ws == 1 else None

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        # faithful configuration: 1 thread (the reference's Eigen GEMV is
        # single-threaded; no OpenMP in proj/CMakeLists.txt)
        rows = max(64, int(2.5e8 // ((spec.n + 3) // 4)))
        gbs, steps, el = cpu_port_sample(W, spec, rows, 1, 10.0)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "port",
               "sample": f"oracle packed operator (1 thread), apply+apply_adjoint on SNPs "
                         f"[0,{rows}) of config {cfg}, {steps} steps in {el:.1f}s"}
        if not args.no_cpu_svdl:
            # time to solution on the reference's literal dense path (config 1),
            # beside the GPU solve of the same config
            sv = cpu_dense_svdl(W, 1)
            op1 = gkb.GenotypeOperator.from_synth(synth.config_spec(1), ctx=ctx,
                                                  scheme=gkb.ScalingScheme.kHwe)
            o1 = synth.config_options(1)
            gkb.svdl(op1, o1)
            t0 = time.perf_counter()
            r1 = gkb.svdl(op1, o1)
            sv["gpu_seconds"] = round(time.perf_counter() - t0, 4)
            sv["gpu_mvps"] = r1.stats.mvps
            sv["gpu_sigma_1"] = float(r1.singvals[0])
            op1.close()
            cpu["svdl"] = sv

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 5),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based generator of the config's BASELINE model, "
                    "device-generated)",
            "config": config_block(W, cfg, spec, ws),
            "gpu_launches": launches * args.steps,
            "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": round(dom[1], 1),
                         "peak": peak, "unit": "GB/s", "frac": round(dom[1] / peak, 4),
                         "traffic": traffic[0] if traffic else None,
                         "traffic_source": f"profiles/{traffic[1]} (dram read+write per launch)"
                         if traffic else None,
                         "peak_source": peak_src,
                         "k1_apply_gbs": round(k1_gbs, 1), "k2_adjoint_gbs": round(k2_gbs, 1),
                         "k1_main_ms": round(k1_main, 5), "k2_main_ms": round(k2_main, 5),
                         "k1_step_ms": round(k1_ms, 5), "k2_step_ms": round(k2_ms, 5),
                         "algorithmic_bytes_per_launch": b_mvp},
            "e2e": {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "time_to_solution": {"seconds": round(tts, 4), "device_seconds":
                                 round(res.stats.device_seconds, 4), "mvps": res.stats.mvps,
                                 "steps": res.stats.steps, "restarts": res.stats.restarts,
                                 "converged": res.stats.converged, "k": opts.k,
                                 "host_syncs": res.stats.host_syncs,
                                 "solve_gbs": round(res.stats.mvps * packed_total / tts / 1e9, 1),
                                 "first_call_seconds": round(tts_first, 4),
                                 "note": "second solve on the same operator; the first call also "
                                         "allocates the solver's device/pinned buffers",
                                 "options": W.OPTIONS_TEXT[cfg]},
            "clocks": clocks,
            "build_seconds": round(t_build, 3),
        }
        if ingest:
            line["ingest"] = ingest
        if widened:
            line["widened"] = widened
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CFG, choices=[1, 2, 3, 4])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-cpu-svdl", action="store_true",
                    help="skip the CPU time-to-solution leg (config 1, dense, 1 thread)")
    ap.add_argument("--no-ingest", action="store_true", help="skip the .bed ingest timing")
    ap.add_argument("--no-widen", action="store_true",
                    help="skip the subspace / regression timings")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
