#!/usr/bin/env python3
"""Benchmark of the B200 kNN-interaction operator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5] [--scaling strong|weak] [--launch graph|stream]

Workload (default, BASELINE.json configs[1] "C2"): N = 1,000,000 points in
D = 49 from the 3-level mixture, exact kNN k = 30, Gaussian weights
exp(-d^2/h^2) with h the median kNN distance, x ~ U[0,1]; one step = one
application y = A x of the cluster-ordered operator (30,000,000
interactions).  Inputs (values 120 MB + 16-bit indices 60 MB) exceed the
126 MB L2, so no flush is needed between steps.

Multi-GPU (torchrun, one process per GPU, NCCL): the cluster-ordered rows are
cut into N contiguous, tile-aligned row blocks balanced by nonzeros (strong
scaling); x is replicated and the fixed-charge iteration has
no exchange.  --scaling weak gives rank r its own seeded instance instead.

--impl reference times the reference's own CPU path on the same config
(oracle/refbench.py): the UNMODIFIED patchord library (oracle/_ref) builds
its own ordering and hierarchy from inputs made without the product library
(libknnx.so is never loaded in that arm) and runs spmv_hier_parallel with
every host thread, one call per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# BASELINE.json metric; the step (C2 y = A x, C3 mean shift, ...) is named in config.workload
METRIC = "kNN interaction nnz/sec and achieved HBM GB/s vs roofline"

# config.workload text per BASELINE config (identical in both arms)
WORK = {
    "c1": "original + cluster-ordered y=Ax",
    "c2": "cluster-ordered y=Ax",
    "c3": "mean shift step (weights recomputed, SpMM with D right-hand sides)",
    "c4": "t-SNE attractive step with embedding update",
    "c5": "Gaussian-recompute y=A(t,s)x",
}
SHAPES = {"c1": (20_000, 49, 30), "c2": (1_000_000, 49, 30), "c3": (1_000_000, 49, 30),
          "c4": (4_000_000, 50, 90), "c5": (1_000_000, 960, 16)}


def log(msg: str) -> None:
    print(msg, file=sys.stderr, flush=True)


def config_dict(name: str, n: int | None = None) -> dict:
    """The config object both arms print (same keys, same values)."""
    n0, dim, k = SHAPES[name[:2]]
    n = n or n0
    return {"workload": f"{name[:2]}: {WORK[name[:2]]}, N={n}, D={dim}, k={k}", "n": n, "dim": dim,
            "k": k}


def peaks() -> dict:
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def golden_perm(name: str) -> str | None:
    """sha256 of the reference's make_ordering("tree3") permutation at the
    config's full size (tests/golden/perm_hashes.json, made by the reference)."""
    p = os.path.join(HERE, "tests", "golden", "perm_hashes.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        rec = json.load(f).get({"c3": "c2"}.get(name, name))
    return rec["sha256"] if rec else None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    """One process per GPU over NCCL.  KNNX_BENCH_FUNCTIONAL=1 (test switch,
    never for numbers): gloo and ranks folded onto the visible devices, so the
    N > 1 code path can be exercised on a one-GPU box -- its ranks never wait
    on each other's kernels."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    functional = os.environ.get("KNNX_BENCH_FUNCTIONAL", "0") == "1"
    if functional:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


def alg_bytes_csr(nnz: int, m: int, n: int) -> int:
    """SURVEY.md §8d stationary basis: 8 nnz + 4 (M+1) + 4 N + 4 M."""
    return 8 * nnz + 4 * (m + 1) + 4 * n + 4 * m


def format_bytes(info: dict) -> int:
    """Compulsory bytes of the 16-bit cluster-tile format per launch."""
    stored = info["stored"]
    slices = (info["n_rows"] + 31) // 32
    return (4 * stored + 2 * stored + 4 * info["halo_total"] + 8 * (info["n_tiles"] + 1)
            + 12 * slices + 4 * info["n_cols"] + 4 * info["n_rows"])


def traffic_of(kernel_key: str):
    p = os.path.join(HERE, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(kernel_key)
    return None


# ---------------------------------------------------------------------------
# reference arm


def run_reference(args, world: int) -> None:
    """--impl reference: the reference CPU path on this host (rank 0 only),
    inputs built without the product library (oracle/refbench.py)."""
    from oracle import refbench
    name = args.config[:2]
    if name == "c2" or name == "c1":
        n = args.n or SHAPES[name][0]
        r = refbench.run_c2(args.steps, args.warmup, n=n, log=log)
        value = r["value"]
        line = {
            "metric": METRIC, "value": value, "unit": "interactions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": args.scaling if world > 1 else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded 3-level mixture, exact kNN, Gaussian weights)",
            "config": config_dict(name, n), "impl": "reference",
            "parallelism": f"spmv_hier_parallel, {r['workers']} host threads",
            "cpu_baseline": {
                "value": value, "unit": "interactions/s", "cores": r["workers"], "kind": "reference",
                "sample": (f"spmv_hier_parallel({r['workers']} workers) per step over the full "
                           f"C2 matrix (nnz {r['nnz']}), cut level {r['cut_level']}; the "
                           "reference's own make_ordering(tree3) + build_hier on inputs built "
                           "by the oracle (no product library)"),
                "host": r["host"], "median_value": r["median_value"],
                "spmv_hier_1thread": r["spmv_hier_1thread"]},
            "e2e": {"value": value, "unit": "interactions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "checks": {"permutation_sha256": r["permutation_sha256"],
                       "permutation_matches_golden": (r["permutation_sha256"] == golden_perm(name)
                                                      if n == SHAPES[name][0] else None),
                       "h": r["h"], "pca_iterations": r["pca_iterations"]},
            "setup_s": r["setup_s"],
        }
    else:
        r = refbench.run_nonstationary(name, log=log)
        line = {
            "metric": METRIC, "value": r["value"], "unit": "interactions/s", "n_gpus": world,
            "steps": 3, "warmup": 0, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mixture, exact kNN)", "config": config_dict(name),
            "impl": "reference", "parallelism": "single thread (the reference has no parallel "
                                                "non-stationary kernels)",
            "cpu_baseline": {"value": r["value"], "unit": "interactions/s", "cores": 1,
                             "kind": "reference", "sample": r["sample"], "host": r["host"]},
            "e2e": {"value": r["value"], "unit": "interactions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# CPU baselines inside our arm (reference code on our workload, rank 0, N=1)


def reference_cpu_baseline(wl, budget_s: float = 12.0) -> dict:
    """patchord's own spmv_hier_parallel on this host over our C2 graph; the
    reference builds its hierarchy from our tree embedding (oracle/_ref)."""
    from oracle import refbench
    from oracle.oracle import Ref, RefHier
    ref = Ref()
    hw = ref.hardware_threads()
    rp_o, cols_o, vals_o = wl.csr_o.export()
    t0 = time.perf_counter()
    h, fwd = RefHier.from_original(ref, rp_o, cols_o, vals_o.astype(np.float64), wl.embedding)
    build_s = time.perf_counter() - t0
    xc = np.empty(wl.cfg.n)
    xc[fwd] = wl.x.astype(np.float64)
    _, t1 = h.bench(xc, hw, 1)
    reps = int(max(3, min(41, budget_s / max(t1[0] * 1e-9, 1e-6))))
    _, times = h.bench(xc, hw, reps)
    med = float(np.median(times)) * 1e-9
    _, ts = h.bench(xc, 0, 3)
    nnz = wl.nnz
    return {
        "value": nnz / med, "unit": "interactions/s", "cores": hw, "kind": "reference",
        "sample": f"C2 full matrix, spmv_hier_parallel({hw} workers), median of {reps} reps "
                  f"(+1 warm-up), reference built -O3 no -march",
        "spmv_hier_1thread": nnz / (float(np.median(ts)) * 1e-9),
        "ref_build_s": round(build_s, 2), "cut_level": h.info()["cut_level"],
        "host": refbench.host_cpu(ref),
    }


def nonstat_cpu_baseline(cfg, wl, n_rows: int) -> dict:
    """The reference's own non-stationary CPU path (oracle/_ref, single
    thread: the reference has no parallel versions) on a bounded sample of the
    config: the first `n_rows` cluster-ordered targets with the sources their
    rows reference relabelled compactly (same per-interaction work).
    C3 meanshift_step, C4 tsne_attractive_step (principal submatrix, flat
    HierBlockMatrix), C5 iterate_interactions with the Gaussian value model
    (update_values + spmv_hier per iteration); median of 3 calls, each timed
    around the reference call only."""
    from oracle import refbench
    from oracle.oracle import Oracle, Ref, RefHier
    ref = Ref()
    rp, cols, vals = wl.csr_c.export()
    e1 = int(rp[n_rows])
    if cfg.name.startswith("c4"):
        r = np.repeat(np.arange(n_rows), np.diff(rp[:n_rows + 1]))
        c = cols[:e1]
        keep = c < n_rows
        cnt = np.bincount(r[keep], minlength=n_rows)
        srp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        h = RefHier.flat(ref, n_rows, n_rows, srp, c[keep], vals[:e1][keep].astype(np.float64))
        y0 = Oracle().rng_normal(2, 2 * n_rows).reshape(n_rows, 2) * 1e-2
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            h.tsne(y0)
            times.append(time.perf_counter() - t0)
        nnz = int(keep.sum())
        what = (f"tsne_attractive_step on the principal {n_rows}-row submatrix of the "
                f"cluster-ordered P ({nnz} entries)")
    else:
        uniq, inv = np.unique(cols[:e1], return_inverse=True)
        src = wl.points_c[uniq].astype(np.float64)
        tgt = wl.points_c[:n_rows].astype(np.float64)
        nnz = e1
        if cfg.name.startswith("c3"):
            ids = inv.reshape(n_rows, cfg.k).astype(np.int32)
            times = list(ref.bench_meanshift(src, tgt, ids, wl.h_ref, 3) * 1e-9)
            what = f"meanshift_step for the first {n_rows} targets ({nnz} interactions)"
        else:
            srp = rp[:n_rows + 1].astype(np.int64)
            h = RefHier.flat(ref, n_rows, uniq.size, srp, inv.astype(np.int32), np.ones(nnz))
            xs = np.tile(wl.x_c[uniq].astype(np.float64), (3, 1))
            _, t_ns = h.iterate_gaussian(tgt, src, wl.h_ref, xs)
            times = list(t_ns * 1e-9)
            what = (f"iterate_interactions (Gaussian update_values + spmv_hier) for the first "
                    f"{n_rows} rows ({nnz} interactions, D={cfg.dim})")
    med = float(np.median(times))
    return {"value": nnz / med, "unit": "interactions/s", "cores": 1, "kind": "reference",
            "sample": what + ", median of 3, reference built -O3 no -march",
            "host": refbench.host_cpu(ref)}


# ---------------------------------------------------------------------------
# full-size parity checks (after the timed region)


def sample_rows(n: int, m: int = 2048) -> np.ndarray:
    """m rows spread over the whole operator (seeded), sorted."""
    rng = np.random.default_rng(12345)
    return np.sort(rng.choice(n, min(m, n), replace=False))


def sub_csr(rp, cols, rows):
    """Rows `rows` of a CSR with their columns relabelled compactly."""
    lens = rp[rows + 1] - rp[rows]
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    c = cols[idx]
    uniq, inv = np.unique(c, return_inverse=True)
    srp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return srp, inv.astype(np.int32), uniq, idx


def spmv_rows_check(wl, y_c: np.ndarray, rows: np.ndarray) -> float:
    """C2: sampled rows of the GPU y against the double oracle on identical
    fp32 inputs (values as stored, x widened); scale-aware metric."""
    from oracle.oracle import Oracle, scale_rel
    rp, cols, vals = wl.csr_c.export()
    srp, scols, uniq, idx = sub_csr(rp, cols, rows)
    want = Oracle().spmv(srp, scols, vals[idx].astype(np.float64), wl.x_c[uniq].astype(np.float64))
    return float(scale_rel(y_c[rows], want))


def meanshift_rows_oracle(wl, cfg, rows, t_rows: np.ndarray) -> np.ndarray:
    """One oracle meanshift_step for targets `rows` at positions t_rows
    (sources fixed = the initial points)."""
    from oracle.oracle import Oracle
    rp, cols, _ = wl.csr_c.export()
    srp, scols, uniq, _ = sub_csr(rp, cols, rows)
    return Oracle().meanshift_step(scols.reshape(len(rows), cfg.k), t_rows.astype(np.float64),
                                   wl.points_c[uniq].astype(np.float64), wl.h_ref)


def gauss_rows_check(wl, cfg, y: np.ndarray, rows) -> float:
    from oracle.oracle import Oracle, scale_rel
    rp, cols, _ = wl.csr_c.export()
    srp, scols, uniq, _ = sub_csr(rp, cols, rows)
    pts = wl.points_c
    want = Oracle().gauss_spmv(srp, scols, pts[rows].astype(np.float64),
                               pts[uniq].astype(np.float64), wl.h_ref,
                               wl.x_c[uniq].astype(np.float64))
    return float(scale_rel(y[rows], want))


def tsne_rows_check(wl, rows, y_full: np.ndarray, f: np.ndarray) -> float:
    """C4: forces of sampled rows from the embedding y_full (n x 2) against the
    direct-form double oracle (pinned to the reference, tests/test_golden.py)."""
    from oracle.oracle import Oracle, scale_rel
    rp, cols, p = wl.csr_c.export()
    lens = rp[rows + 1] - rp[rows]
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    srp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    # direct form over the sampled rows: y_i first, then every y_j
    m = len(rows)
    yy = np.concatenate([y_full[rows], y_full]).astype(np.float64)
    want = Oracle().tsne_rows(srp, (cols[idx] + m).astype(np.int32), p[idx].astype(np.float64),
                              yy, m)
    return float(scale_rel(f[rows], want))


# ---------------------------------------------------------------------------
# our arm: stationary (C1 / C2)


def run_stationary(args, cfg, wl, ctx, stream, world, rank, dev, weak):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import check, lib
    from paper_1709_03671_b200.distributed import partition_rows

    rp_c, _, _ = wl.csr_c.export()
    if world > 1 and not weak:  # nnz-balanced, tile-aligned row block of the one operator
        r0, r1 = partition_rows(rp_c, world, 256)[rank]
    else:
        r0, r1 = 0, cfg.n
    csr_local = wl.csr_c.row_block(r0, r1) if (world > 1 and not weak) else wl.csr_c
    op = api.Operator.from_host_csr(ctx, csr_local, api.CLUSTER)
    info = op.info
    x = torch.from_numpy(wl.x_c).to(f"cuda:{dev}")
    y = torch.empty(r1 - r0, dtype=torch.float32, device=f"cuda:{dev}")

    def timed(fn):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms

    def stream_steps():
        for _ in range(args.steps):
            op.spmv(x, y)

    def graph_steps():  # the K steps as one CUDA-graph replay (knnx_spmv_batch_strided_dev)
        op.spmv_repeat(args.steps, x, y)

    # L2 rule: a rank whose operator + x fit in the 126 MB L2 (row blocks at
    # N >= 2) would re-read them from L2 every step; then the L2 is flushed
    # (a 256-MB memset) before every step and only the steps are timed, each
    # on its own pair of CUDA events
    L2_BYTES = 126 * 2 ** 20
    rank_bytes = format_bytes(info)
    flush = rank_bytes < L2_BYTES
    l2_note = (f"per-rank inputs ({rank_bytes / 1e6:.0f} MB stored) exceed the 126 MB L2; no flush"
               if not flush else
               f"per-rank inputs ({rank_bytes / 1e6:.0f} MB stored) fit the 126 MB L2: a 256-MB "
               "memset flushes it before every step and each step is timed alone (events around "
               "the kernel, stream launches)")
    scrub = torch.empty(64 * 2 ** 20, dtype=torch.float32, device=f"cuda:{dev}") if flush else None

    def flushed_steps():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for e0, e1 in evs:
            scrub.zero_()
            e0.record(stream)
            op.spmv(x, y)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms

    for _ in range(args.warmup):
        op.spmv(x, y)
    graph_steps()  # instantiates the graph (kept on the operator)
    torch.cuda.synchronize()
    launches0 = ctx.launches
    main_fn, other_fn = (graph_steps, stream_steps) if args.launch == "graph" else (stream_steps, graph_steps)
    with ClockSampler(dev) as clk:
        ms = flushed_steps() if flush else timed(main_fn)
    launches = ctx.launches - launches0
    ms_other = timed(other_fn)
    ctx.sync()
    nnz_total = wl.nnz
    if weak:  # every rank processed its own instance of the same shape
        t = torch.tensor([nnz_total], dtype=torch.int64, device=f"cuda:{dev}")
        dist.all_reduce(t)
        nnz_total = int(t.item())
    value = nnz_total * args.steps / (ms * 1e-3)
    per_launch_s = ms * 1e-3 / args.steps

    pk = peaks()
    ab = alg_bytes_csr(info["nnz"], info["n_rows"], info["n_cols"])
    fb = format_bytes(info)
    achieved = ab / per_launch_s / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"],
                "traffic": traffic_of("spmv_tiles_g_kernel") if world == 1 else None,
                "peak_source": pk["source"], "alg_bytes_per_launch": ab,
                "basis": "SURVEY.md §8d CSR basis 8nnz+4(M+1)+4N+4M (per rank)",
                "format_bytes_per_launch": fb,
                "achieved_format_gbs": fb / per_launch_s / 1e9,
                "frac_format": fb / per_launch_s / 1e9 / pk["hbm_gbs"],
                "kernel": "spmv_tiles_g_kernel<4, pdl>", "launch_us": per_launch_s * 1e6}

    extra = {(f"{'stream' if args.launch == 'graph' else 'graph'}_launch" if not flush
              else f"{'stream' if args.launch == 'graph' else 'graph'}_launch_l2_warm"): {
        "launch_us": ms_other * 1e3 / args.steps,
        "value": nnz_total * args.steps / (ms_other * 1e-3)}}
    checks = {}
    y_dev = y.cpu().numpy()
    if world == 1:
        # full-size parity: sampled rows against the double oracle, and the
        # ordering against the reference's own permutation hash
        from oracle import refbench
        checks["oracle_rows_rel"] = spmv_rows_check(wl, y_dev, sample_rows(cfg.n))
        checks["oracle_rows"] = "2048 seeded rows spread over the operator"
        sha = refbench.perm_sha(wl.forward)
        gold = golden_perm(cfg.name) if cfg.n == SHAPES[cfg.name[:2]][0] else None
        checks["permutation_sha256"] = sha
        checks["permutation_matches_reference"] = (sha == gold) if gold else None
        # original-order operator (the spmv_flat path) for comparison
        op_o = api.Operator.from_host_csr(ctx, wl.csr_o, api.ORIGINAL)
        x_o = torch.from_numpy(wl.x).to(f"cuda:{dev}")
        y_o = torch.empty(cfg.n, dtype=torch.float32, device=f"cuda:{dev}")
        for _ in range(args.warmup):
            op_o.spmv(x_o, y_o)

        def orig_steps():
            for _ in range(args.steps):
                op_o.spmv(x_o, y_o)
        ms_o = timed(orig_steps)
        extra["original_order"] = {
            "value": nnz_total * args.steps / (ms_o * 1e-3), "unit": "interactions/s",
            "launch_us": ms_o * 1e3 / args.steps, "kernel": "spmv_orig_kernel",
            "achieved_gbs": ab / (ms_o * 1e-3 / args.steps) / 1e9}
        y_oo = y_o.cpu().numpy()
        checks["cluster_vs_original_rel"] = float(
            np.max(np.abs(y_dev[wl.forward] - y_oo)) / np.max(np.abs(y_oo)))
        op_o.close()

    # end to end through the C ABI with host buffers (H2D x, kernel, D2H y per
    # step), on every rank; whole-job value = all ranks' interactions / the
    # slowest rank's wall time (barrier before each timed call)
    m_loc = r1 - r0

    def wall_max(fn):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        fn()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return el

    xs = torch.from_numpy(np.tile(wl.x_c, (args.e2e_steps, 1))).pin_memory()
    ys = torch.empty(args.e2e_steps, m_loc, dtype=torch.float32).pin_memory()

    def batch():
        check(lib.knnx_spmv_host_batch(op.h, args.e2e_steps, C.c_void_p(xs.data_ptr()),
                                       C.c_void_p(ys.data_ptr())))

    batch()
    elb = sorted(wall_max(batch) for _ in range(3))[1]
    checks["e2e_batch_matches_device"] = bool(np.array_equal(ys[-1].numpy(), y_dev))
    xh, yh = xs[0], torch.empty(m_loc, dtype=torch.float32).pin_memory()

    def unbatched():
        for _ in range(args.e2e_steps):
            check(lib.knnx_spmv_host(op.h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr())))

    unbatched()
    el = wall_max(unbatched)
    checks["e2e_matches_device"] = bool(np.array_equal(yh.numpy(), y_dev))
    # pageable numpy buffers (what a caller holding plain arrays passes)
    xs_p = np.ascontiguousarray(np.tile(wl.x_c, (args.e2e_steps, 1)))
    ys_p = np.empty((args.e2e_steps, m_loc), np.float32)

    def batch_pageable():
        check(lib.knnx_spmv_host_batch(op.h, args.e2e_steps, C.c_void_p(xs_p.ctypes.data),
                                       C.c_void_p(ys_p.ctypes.data)))

    batch_pageable()
    elp = wall_max(batch_pageable)
    checks["e2e_pageable_matches_device"] = bool(np.array_equal(ys_p[-1], y_dev))
    rows_total = cfg.n * world if weak else cfg.n
    e2e = {"value": nnz_total * args.e2e_steps / elb, "unit": "interactions/s",
           "h2d_bytes_per_step": 4 * cfg.n * world, "d2h_bytes_per_step": 4 * rows_total,
           "steps": args.e2e_steps,
           "api": "knnx_spmv_host_batch (C ABI, pinned host buffers: x by copy engine, y stored "
                  "by the multiply into the caller's buffer), median of 3 calls",
           "unbatched_value": nnz_total * args.e2e_steps / el,
           "unbatched_api": "knnx_spmv_host per step (pinned)",
           "pageable_value": nnz_total * args.e2e_steps / elp,
           "pageable_api": "knnx_spmv_host_batch with pageable numpy buffers (copy engines)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_cpu_baseline(wl)
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "interactions/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "interactions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if weak else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded 3-level mixture, exact device kNN, Gaussian weights)"
                    + ("; weak scaling: rank r owns instance seed=16r" if weak else ""),
            "config": config_dict(cfg.name, cfg.n),
            "parallelism": (f"independent instances x{world}" if weak
                            else f"row-block x{world} (nnz-balanced, tile-aligned; x replicated)"),
            "launch": ("stream launches, one timed step each (L2 flushed between steps)" if flush else
                       f"{args.launch} ({'one CUDA-graph replay of the K steps' if args.launch == 'graph' else 'K stream launches'}, PDL)"),
            "l2": l2_note,
            "nnz": nnz_total, "tile_rows": info["tile_rows"],
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "extra": extra, "checks": checks,
            "setup_s": {k: (round(v, 2) if isinstance(v, float) else v) for k, v in wl.timings.items()},
        }
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm: non-stationary (C3 / C4 / C5)


def run_nonstationary(args, cfg, wl, ctx, stream, world, rank, dev):
    """C3 (mean shift, D=49, k=30 incl. self), C4 (t-SNE attraction, k=90
    symmetrised P) and C5 (Gaussian recompute, D=960) on row-block shards; C3
    publishes the moved targets with an all-gather on a side stream (nothing
    in the next step waits on it), C4 all-gathers the embedding every
    iteration (the next step needs it), C5 has no exchange (x fixed)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import check, lib
    from paper_1709_03671_b200.distributed import RowGather, ShardedOperator

    # C3/C4 on int32 columns over the tree-ordered rows ("flat": one dependent
    # load per neighbour instead of two; C4 N=1M 0.76 vs 0.89 ms, C3 564 vs
    # 596 us); C3-C5 rows in the graph-locality schedule (C4 N=1M 760 -> 695 us);
    # C4 entries group-interleaved for the 8-lane t-SNE groups (699 -> 561 us)
    name = cfg.name[:2]
    layout = api.ORIGINAL if name in ("c3", "c4") else None
    opts = api.OPT_GROUP_INTERLEAVE if name == "c4" else 0
    t_op = time.perf_counter()
    dev_csr = getattr(wl, "dev_csr", None)
    sop = ShardedOperator(ctx, wl.csr_c, world, rank, tile_rows=256, layout=layout,
                          schedule=True, options=opts, dev_csr=dev_csr)
    if dev_csr is not None:  # C4: the operator (or this rank's row block) was built on the device
        dev_csr.free()
        wl.dev_csr = None
        wl.timings["operator_build"] = "device (knnx_op_create_csr_dev)"
    wl.timings["operator_s"] = time.perf_counter() - t_op
    r0, r1 = sop.rows
    info = sop.op.info
    n, D = cfg.n, cfg.dim
    nnz_local = info["nnz"]
    nnz_total = wl.nnz
    side = torch.cuda.Stream(dev)
    extra: dict = {}
    checks: dict = {}
    e2e = None
    if name == "c3":
        s = api.to_device_points(wl.points_c, f"cuda:{dev}")
        bufs = [s.clone(), s.clone()]
        h = wl.h_ref
        gathered = [torch.cuda.Event(), torch.cuda.Event()]
        gather = RowGather(sop.shard, (s.shape[1],), s.dtype, s.device, ctx, sop.group)
        state = {"i": 0}

        def step():
            a, b = bufs[state["i"] & 1], bufs[(state["i"] + 1) & 1]
            if world > 1:  # b's previous gather must have read our rows
                stream.wait_event(gathered[(state["i"] + 1) & 1])
            sop.op.meanshift(a[r0:r1], s, D, h, b[r0:r1])
            if world > 1:
                ev = torch.cuda.Event()
                ev.record(stream)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    gather(b[r0:r1], b)
                gathered[(state["i"] + 1) & 1].record(side)
            state["i"] += 1

        alg = 4 * D * n + 8 * D * (r1 - r0) + 4 * nnz_local + 4 * (r1 - r0 + 1)
        kernel = "meanshift_lane_kernel<G=8, NB=2, 64 regs> (int32 ids, graph schedule)"
        tkey = "meanshift_lane_kernel"
    elif name == "c5":
        s = api.to_device_points(wl.points_c, f"cuda:{dev}")
        x = torch.from_numpy(wl.x_c).to(f"cuda:{dev}")
        y = torch.empty(r1 - r0, device=f"cuda:{dev}")
        h = wl.h_ref

        def step():
            sop.op.gauss_spmv(s[r0:r1], s, D, h, x, y)

        rp_l, cols_l, _ = wl.csr_c.row_block(r0, r1).export() if world > 1 else wl.csr_c.export()
        # coordinates of the distinct points touched, read once
        # (targets and sources are the same point set), + ids + row_ptr + x + y
        n_distinct = int(np.union1d(np.unique(cols_l), np.arange(r0, r1)).size)
        n_src = int(np.unique(cols_l).size)
        alg = 4 * D * n_distinct + 4 * nnz_local + 4 * (r1 - r0 + 1) + 4 * n_src + 4 * (r1 - r0)
        kernel = "gauss_warp_kernel<tiles, 8> (warp per row, FFMA2, D=960, graph schedule)"
        tkey = "gauss_warp_kernel"
    else:
        y0 = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)  # y_i ~ N(0, 1e-4 I)
        ybuf = [torch.from_numpy(y0[wl.inverse]).to(f"cuda:{dev}"),
                torch.zeros(n, 2, device=f"cuda:{dev}")]
        f = torch.empty(r1 - r0, 2, device=f"cuda:{dev}")
        ynew = torch.empty(r1 - r0, 2, device=f"cuda:{dev}")
        eta = 4.0 * n / 12.0  # y <- y - eta * F (gradient 4F, learning rate N/12)
        state = {"i": 0}
        fused = world > 1 and args.exchange == "fused"
        if fused:  # peer stores into every rank's replica + NCCL barrier
            sop.enable_fused_tsne(ybuf)

        def step():
            a, b = ybuf[state["i"] & 1], ybuf[(state["i"] + 1) & 1]
            if fused:
                sop.tsne_step_fused(a, 2, f, eta, (state["i"] + 1) & 1)
            elif world > 1:
                sop.tsne_step(a, 2, f, eta, ynew, b)
            else:
                sop.op.tsne(a, 2, f, False, eta, b)
            state["i"] += 1

        alg = 8 * nnz_local + 4 * (r1 - r0 + 1) + 8 * n + 8 * (r1 - r0) + 8 * (r1 - r0)
        kernel = "tsne_group_kernel<G=8, interleaved, 40 regs> (fused F + y update, int32 ids)"
        tkey = "tsne_group_kernel_interleaved"

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ctx.launches
    with ClockSampler(dev) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        stream.wait_stream(side)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctx.sync()
    launches = ctx.launches - launches0
    per = ms * 1e-3 / args.steps
    pk = peaks()
    roofline = {"bound": "hbm", "achieved": alg / per / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": alg / per / 1e9 / pk["hbm_gbs"],
                "traffic": traffic_of(tkey) if world == 1 else None,
                "peak_source": pk["source"], "alg_bytes_per_launch": alg, "kernel": kernel,
                "launch_us": per * 1e6, "basis": "SURVEY.md §8d (per rank)"}

    if world == 1 and not args.no_checks:
        rows = sample_rows(n)
        if name == "c3":
            # teacher forcing over the config's 20 iterations: every GPU step
            # against one oracle step from the GPU's previous positions; drift
            # = the GPU trajectory against the oracle's own (free-running)
            # trajectory of the same targets (sources fixed, rows independent)
            rows_t = torch.from_numpy(rows).to(f"cuda:{dev}")
            cur = s.clone()
            nxt = torch.empty_like(s)
            free = wl.points_c[rows].astype(np.float64)
            tf, drift = [], []
            from oracle.oracle import scale_rel
            for _ in range(cfg.iterations):
                sop.op.meanshift(cur, s, D, h, nxt)
                ctx.sync()
                got = nxt.index_select(0, rows_t)[:, :D].cpu().numpy()
                prev = cur.index_select(0, rows_t)[:, :D].cpu().numpy()
                tf.append(float(scale_rel(got, meanshift_rows_oracle(wl, cfg, rows, prev))))
                free = meanshift_rows_oracle(wl, cfg, rows, free)
                drift.append(float(scale_rel(got, free)))
                cur, nxt = nxt, cur
            checks["oracle_rows_rel"] = tf[0]
            checks["teacher_forced_rel_per_step"] = tf
            checks["teacher_forced_max"] = max(tf)
            checks["drift_rel_per_step"] = drift
            checks["rows"] = f"{len(rows)} seeded rows, {cfg.iterations} steps"
        elif name == "c5":
            step()
            ctx.sync()
            checks["oracle_rows_rel"] = gauss_rows_check(wl, cfg, y.cpu().numpy(), rows)
            checks["rows"] = f"{len(rows)} seeded rows"
            # size-independent property over all rows: the operator is linear
            # in the charge, A(x + x') = A x + A x' to fp32 rounding
            x2 = torch.rand(n, device=x.device, generator=torch.Generator(device=x.device).manual_seed(5))
            y1, y2, y12 = y.clone(), torch.empty_like(y), torch.empty_like(y)
            sop.op.gauss_spmv(s[r0:r1], s, D, h, x2, y2)
            sop.op.gauss_spmv(s[r0:r1], s, D, h, x + x2, y12)
            ctx.sync()
            checks["linearity_rel"] = float(((y1 + y2 - y12).abs().max() / y12.abs().max()).item())
        else:
            # teacher forcing over the config's 50 iterations: forces of the
            # sampled rows from the GPU's current embedding vs the oracle
            ya = torch.from_numpy(y0[wl.inverse]).to(f"cuda:{dev}")
            yb = torch.empty_like(ya)
            f1 = torch.empty(n, 2, device=f"cuda:{dev}")
            tf = []
            for it in range(cfg.iterations):
                sop.op.tsne(ya, 2, f1, False, eta, yb)
                ctx.sync()
                tf.append(tsne_rows_check(wl, rows, ya.cpu().numpy(), f1.cpu().numpy()))
                ya, yb = yb, ya
            checks["oracle_rows_rel"] = tf[0]
            checks["teacher_forced_rel_per_step"] = tf
            checks["teacher_forced_max"] = max(tf)
            checks["rows"] = f"{len(rows)} seeded rows, {cfg.iterations} steps"
            # size-independent properties of the device-built P (the reference's
            # symmetrize + normalisation, knn.cpp:72-84): sums to 1, symmetric
            # on sampled entries, and holds every kNN edge of sampled rows
            prp, pcols, pvals = wl.csr_c.export()
            checks["p_sum"] = float(np.sum(pvals, dtype=np.float64))
            rs = np.random.default_rng(7)
            ent = rs.integers(0, pcols.size, 20000)
            ri = np.searchsorted(prp, ent, side="right") - 1
            ci = pcols[ent].astype(np.int64)
            lo, hi = prp[ci], prp[ci + 1]
            pos = np.array([lo[q] + np.searchsorted(pcols[lo[q]:hi[q]], ri[q]) for q in range(ent.size)])
            ok = (pos < hi) & (pcols[np.minimum(pos, pcols.size - 1)] == ri)
            checks["p_symmetric_sampled"] = bool(ok.all() and np.array_equal(pvals[pos[ok]], pvals[ent[ok]]))
            held = all(np.isin(wl.knn_ids_c[r], pcols[prp[r]:prp[r + 1]]).all() for r in rows[:512])
            checks["p_holds_knn_edges_sampled"] = bool(held)
        sha = refbench_sha(wl.forward)
        gold = golden_perm(name) if cfg.n == SHAPES[name][0] else None
        checks["permutation_sha256"] = sha
        checks["permutation_matches_reference"] = (sha == gold) if gold else None

    if world == 1 and not args.no_e2e:
        # end to end through the host-buffer C ABI (pinned buffers): every
        # step copies its inputs in and its result out
        steps = 5
        if name == "c3":
            th = torch.from_numpy(np.ascontiguousarray(wl.points_c)).pin_memory()
            oh = torch.empty_like(th).pin_memory()

            def e2e_step():
                check(lib.knnx_meanshift_host(sop.op.h, C.c_void_p(th.data_ptr()),
                                              C.c_void_p(th.data_ptr()), D, h,
                                              C.c_void_p(oh.data_ptr())))
            hb, db = 2 * 4 * D * n, 4 * D * n
            api_name = "knnx_meanshift_host (targets + sources in, positions out)"
        elif name == "c4":
            yh = torch.from_numpy(np.ascontiguousarray(y0[wl.inverse])).pin_memory()
            fh = torch.empty_like(yh).pin_memory()

            def e2e_step():
                check(lib.knnx_tsne_attr_host(sop.op.h, C.c_void_p(yh.data_ptr()), 2,
                                              C.c_void_p(fh.data_ptr()), 0))
            hb, db = 8 * n, 8 * n
            api_name = "knnx_tsne_attr_host (embedding in, forces out)"
        else:
            th = torch.from_numpy(np.ascontiguousarray(wl.points_c)).pin_memory()
            xh = torch.from_numpy(wl.x_c).pin_memory()
            yh = torch.empty(n, dtype=torch.float32).pin_memory()

            def e2e_step():
                check(lib.knnx_gauss_spmv_host(sop.op.h, C.c_void_p(th.data_ptr()),
                                               C.c_void_p(th.data_ptr()), D, h,
                                               C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr())))
            hb, db = 4 * D * n + 4 * n, 4 * n
            api_name = "knnx_gauss_spmv_host (points once (t == s) + x in, y out)"
        e2e_step()
        t0 = time.perf_counter()
        for _ in range(steps):
            e2e_step()
        el = (time.perf_counter() - t0) / steps
        e2e = {"value": nnz_total / el, "unit": "interactions/s", "h2d_bytes_per_step": hb,
               "d2h_bytes_per_step": db, "steps": steps, "api": api_name + ", pinned buffers"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = nonstat_cpu_baseline(cfg, wl, {"c3": 100_000, "c4": 60_000}.get(name, 4_000))
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "interactions/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": nnz_total * args.steps / (ms * 1e-3), "unit": "interactions/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded mixture, exact device kNN)",
            "config": config_dict(cfg.name, cfg.n), "nnz": nnz_total,
            "parallelism": f"row-block x{world}",
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "checks": checks, "extra": extra,
            "setup_s": {k: (round(v, 2) if isinstance(v, float) else v) for k, v in wl.timings.items()},
        }
        print(json.dumps(line), flush=True)


def refbench_sha(fwd) -> str:
    from oracle import refbench
    return refbench.perm_sha(fwd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n", "--points", dest="n", type=int, default=None, help="override the point count (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-checks", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--launch", default="graph", choices=["graph", "stream"],
                    help="c1/c2 timed steps: one CUDA-graph replay of the K launches (default) "
                         "or K stream launches")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "fused"],
                    help="c4 at N>1: NCCL all-gather of the embedding after the kernel, or the "
                         "fused path (the kernel stores into every rank's replica over "
                         "NVLink through CUDA-IPC mappings, then a stream-ordered barrier)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="c1/c2 at N>1: strong = one instance, row-block sharded with x "
                         "replicated (default); weak = rank r owns the independent seeded "
                         "instance seed=16r (no data-path collective)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        # rank 0 alone times the reference CPU path; no process group, no CUDA
        # and no product library in this arm
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if int(os.environ.get("RANK", "0")) == 0:
            run_reference(args, world)
        return

    import torch
    import torch.distributed as dist
    world, rank, local = dist_setup()

    from paper_1709_03671_b200 import api, workloads
    dev = torch.cuda.current_device()
    ctx = api.Context(dev)
    stream = torch.cuda.Stream(dev)  # one non-default stream for the library and the events
    torch.cuda.set_stream(stream)
    ctx.use_stream(stream)
    cfg = workloads.CONFIGS[args.config] if args.n is None else workloads.scaled(args.config, args.n)
    weak = world > 1 and args.scaling == "weak" and args.config in ("c1", "c2")
    wl = workloads.build(cfg, ctx, dev, with_values=args.config in ("c1", "c2"),
                         log=log if rank == 0 else None, seed=16 * rank if weak else 0,
                         keep_device_csr=args.config == "c4")
    if args.config in ("c3", "c4", "c5"):
        run_nonstationary(args, cfg, wl, ctx, stream, world, rank, dev)
    else:
        run_stationary(args, cfg, wl, ctx, stream, world, rank, dev, weak)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
