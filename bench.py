#!/usr/bin/env python3
"""Benchmark of the B200 kNN-interaction operator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Workload (default, BASELINE.json configs[1] "C2"): N = 1,000,000 points in
D = 49 from the 3-level mixture, exact kNN k = 30, Gaussian weights
exp(-d^2/h^2) with h the median kNN distance, x ~ U[0,1]; one step = one
application y = A x of the cluster-ordered operator (30,000,000
interactions).  Inputs (values 120 MB + 16-bit indices 60 MB) exceed the
126 MB L2, so no flush is needed between steps.  Multi-GPU (torchrun): the
cluster-ordered rows are cut into N contiguous row blocks (strong scaling),
x is replicated, no exchange is needed in the stationary loop.

--impl reference times the reference's own CPU path (patchord
spmv_hier_parallel with every host thread, oracle/_ref built from the
reference sources) on the same workload.
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


def log(msg: str) -> None:
    print(msg, file=sys.stderr, flush=True)


def peaks() -> dict:
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


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
    N > 1 code path of the default (weak-scaling C2) bench can be exercised on
    a one-GPU box -- its ranks never wait on each other's kernels."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    functional = os.environ.get("KNNX_BENCH_FUNCTIONAL", "0") == "1"
    if functional:
        local = local % max(1, torch.cuda.device_count())
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def shard_rows(n_rows: int, world: int, rank: int, granule: int = 256):
    """Contiguous row block of this rank, cut on tile (granule) boundaries."""
    tiles = (n_rows + granule - 1) // granule
    t0 = tiles * rank // world
    t1 = tiles * (rank + 1) // world
    return min(n_rows, t0 * granule), min(n_rows, t1 * granule)


def alg_bytes_csr(nnz: int, m: int, n: int) -> int:
    """SURVEY.md §8d stationary basis: 8 nnz + 4 (M+1) + 4 N + 4 M."""
    return 8 * nnz + 4 * (m + 1) + 4 * n + 4 * m


def format_bytes(info: dict) -> int:
    """Compulsory bytes of the 16-bit cluster-tile format per launch."""
    stored = info["stored"]
    slices = (info["n_rows"] + 31) // 32
    return (4 * stored + 2 * stored + 4 * info["halo_total"] + 8 * (info["n_tiles"] + 1)
            + 12 * slices + 4 * info["n_cols"] + 4 * info["n_rows"])


def reference_cpu_baseline(wl, budget_s: float = 12.0) -> dict:
    """patchord's own CPU path on this host (oracle/_ref), bounded sample."""
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
    from oracle.oracle import Ref, RefHier
    ref = Ref()
    rp, cols, vals = wl.csr_c.export()
    e1 = int(rp[n_rows])
    if cfg.name.startswith("c4"):
        # principal submatrix: entries whose column is inside the sample
        r = np.repeat(np.arange(n_rows), np.diff(rp[:n_rows + 1]))
        c = cols[:e1]
        keep = c < n_rows
        cnt = np.bincount(r[keep], minlength=n_rows)
        srp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        h = RefHier.flat(ref, n_rows, n_rows, srp, c[keep], vals[:e1][keep].astype(np.float64))
        y0 = api_normal_embedding(n_rows)
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
            "sample": what + ", median of 3, reference built -O3 no -march"}


def oracle_rows_check(cfg, wl, got, m: int = 2048) -> float:
    """Full-size parity spot check: the first m cluster-ordered rows of the
    GPU result against the double oracle (C3 mean-shift positions, C5
    Gaussian-recompute y), sources relabelled compactly; scale-aware metric."""
    from oracle.oracle import Oracle, scale_rel
    orc = Oracle()
    rp, cols, _ = wl.csr_c.export()
    e1 = int(rp[m])
    uniq, inv = np.unique(cols[:e1], return_inverse=True)
    src = wl.points_c[uniq].astype(np.float64)
    tgt = wl.points_c[:m].astype(np.float64)
    if cfg.name.startswith("c3"):
        want = orc.meanshift_step(inv.reshape(m, cfg.k).astype(np.int32), tgt, src, wl.h_ref)
        return float(scale_rel(got[:m], want))
    want = orc.gauss_spmv(rp[:m + 1].astype(np.int64), inv.astype(np.int32), tgt, src, wl.h_ref,
                          wl.x_c[uniq].astype(np.float64))
    return float(scale_rel(got[:m], want))


def api_normal_embedding(n: int) -> np.ndarray:
    from paper_1709_03671_b200 import api
    return api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2).astype(np.float64)


def run_reference(args, world, rank):
    """--impl reference: the reference CPU path on this host, timed per step."""
    import torch
    from oracle.oracle import Ref, RefHier
    from paper_1709_03671_b200 import api, workloads
    ctx = api.Context(torch.cuda.current_device())
    cfg = workloads.CONFIGS[args.config] if args.n is None else workloads.scaled(args.config, args.n)
    wl = workloads.build(cfg, ctx, torch.cuda.current_device(), log=log,
                         with_values=args.config in ("c1", "c2"))
    ref = Ref()
    hw = ref.hardware_threads()
    if args.config in ("c3", "c4", "c5"):
        # the reference's non-stationary path (single-threaded in the
        # reference) on the bounded sample of nonstat_cpu_baseline
        cpu = nonstat_cpu_baseline(cfg, wl, {"c3": 100_000, "c4": 60_000}.get(cfg.name[:2], 4_000))
        line = {
            "metric": METRIC, "value": cpu["value"], "unit": "interactions/s", "n_gpus": world,
            "steps": 3, "warmup": 0, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mixture, exact device kNN)",
            "config": {"workload": f"{cfg.name}: N={cfg.n}, D={cfg.dim}, k={cfg.k}", "n": cfg.n},
            "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": "interactions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    rp_o, cols_o, vals_o = wl.csr_o.export()
    h, fwd = RefHier.from_original(ref, rp_o, cols_o, vals_o.astype(np.float64), wl.embedding)
    xc = np.empty(cfg.n)
    xc[fwd] = wl.x.astype(np.float64)
    h.bench(xc, hw, max(1, args.warmup))
    _, times = h.bench(xc, hw, args.steps)
    total = float(times.sum()) * 1e-9
    value = wl.nnz * args.steps / total
    line = {
        "metric": METRIC, "value": value, "unit": "interactions/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak" if (world > 1 and args.scaling == "weak" and args.config in ("c1", "c2"))
                   else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 3-level mixture, exact kNN, Gaussian weights)",
        "config": {"workload": f"{cfg.name}: cluster-ordered y=Ax, N={cfg.n}, D={cfg.dim}, "
                               f"k={cfg.k}, nnz={wl.nnz}", "n": cfg.n, "nnz": wl.nnz},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "interactions/s", "cores": hw, "kind": "reference",
                         "sample": f"spmv_hier_parallel({hw} workers) per step over the full C2 "
                                   f"matrix, cut level {h.info()['cut_level']}"},
        "e2e": {"value": value, "unit": "interactions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_nonstationary(args, cfg, wl, ctx, stream, world, rank, dev):
    """C3 (mean shift, D=49, k=30 incl. self) and C4 (t-SNE attraction, k=90
    symmetrised P) on row-block shards; C3 publishes the moved targets with an
    all-gather on a side stream (nothing in the next step waits on it), C4
    all-gathers the embedding every iteration (the next step needs it)."""
    import torch
    import torch.distributed as dist

    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200.distributed import ShardedOperator, all_gather_rows

    # int32 columns on the tree-ordered rows ("flat") skip the halo indirection:
    # measured faster for C4's ~150-entry symmetrised rows (0.76 vs 0.89 ms at
    # N=1M); the 16-bit cluster tiles stay the default elsewhere
    # C3 (k = 30) too: the lean mean-shift kernel is latency bound and the
    # one-load int32 ids beat the two dependent halo loads (564 vs 596 us)
    lay_env = os.environ.get("KNNX_LAYOUT", "flat" if cfg.name[:2] in ("c3", "c4") else "tiles")
    layout = api.ORIGINAL if lay_env == "flat" else None
    # C4's and C5's neighbourhoods are poorly grouped by the 3-D tree order
    # (C5: a 256-row tile references ~1800 distinct sources, 9% in-tile; C4:
    # 32-row tiles reuse a halo entry 1.6x): their rows run in the
    # graph-locality schedule unless KNNX_SCHEDULE=0 (C4 N=1M: 760 -> 695 us;
    # C3: 770 -> 747 us, tile halos halve)
    sched = cfg.name[:2] in ("c3", "c4", "c5") and os.environ.get("KNNX_SCHEDULE", "1") != "0"
    # C4: entries group-interleaved for the 8-lane t-SNE groups (one 32-B
    # sector per group step instead of two half-used ones; N=1M: 699 -> 561 us;
    # relabelling the columns in schedule order adds nothing on top, 561 us)
    opts = int(os.environ.get("KNNX_TSNE_OPTS", "2" if cfg.name.startswith("c4") and layout == api.ORIGINAL
                              else "0"))
    # KNNX_TILE_ROWS=32 + KNNX_GAUSS_STREAM=1 selects the C5 source-streaming
    # experiment (slower than the warp kernel)
    tile_rows = int(os.environ.get("KNNX_TILE_ROWS", "256"))
    sop = ShardedOperator(ctx, wl.csr_c, world, rank, tile_rows=tile_rows, layout=layout,
                          schedule=sched, options=opts)
    r0, r1 = sop.rows
    info = sop.op.info
    n, D = cfg.n, cfg.dim
    nnz_local = info["nnz"]
    nnz_total = wl.nnz
    side = torch.cuda.Stream(dev)
    extra_c5 = {}
    if cfg.name.startswith("c3"):
        s = api.to_device_points(wl.points_c, f"cuda:{dev}")
        bufs = [s.clone(), s.clone()]
        h = wl.h_ref
        gathered = [torch.cuda.Event(), torch.cuda.Event()]
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
                    all_gather_rows(b[r0:r1], sop.shard, b, sop.group)
                gathered[(state["i"] + 1) & 1].record(side)
            state["i"] += 1

        alg = 4 * D * n + 8 * D * (r1 - r0) + 4 * nnz_local + 4 * (r1 - r0 + 1)
        kernel = f"meanshift_lane_kernel<G=8, NB=2, 64 regs> ({lay_env} layout)"
        work = "mean shift step"
    elif cfg.name.startswith("c5"):
        # Gaussian weights recomputed from the coordinates every iteration
        s = api.to_device_points(wl.points_c, f"cuda:{dev}")
        x = torch.from_numpy(wl.x_c).to(f"cuda:{dev}")
        y = torch.empty(r1 - r0, device=f"cuda:{dev}")
        h = wl.h_ref

        def step():
            sop.op.gauss_spmv(s[r0:r1], s, D, h, x, y)

        rp_l, cols_l, _ = wl.csr_c.row_block(r0, r1).export() if world > 1 else wl.csr_c.export()
        n_src = int(np.unique(cols_l).size)
        # targets + every referenced source row once + columns + row pointers + x + y
        alg = 4 * D * (r1 - r0) + 4 * D * n_src + 4 * nnz_local + 4 * (r1 - r0 + 1) + 4 * n_src \
            + 4 * (r1 - r0)
        kernel = ("gauss_stream_kernel<8, B=8, NBUF=6> (32-row tiles, halo streamed by TMA bulk "
                  "copies through shared memory, D=960)" if tile_rows == 32 and
                  os.environ.get("KNNX_GAUSS_STREAM", "0") != "0"
                  else "gauss_warp_kernel<tiles, 8> (warp per row, FFMA2, D=960)")
        work = "Gaussian-recompute y=A(t,s)x"
        if world == 1:  # size-independent check: original order gives the same y
            op_o = api.Operator.from_host_csr(ctx, wl.csr_o, api.ORIGINAL)
            s_o = api.to_device_points(wl.points, f"cuda:{dev}")
            x_o = torch.from_numpy(wl.x).to(f"cuda:{dev}")
            y_o = torch.empty(n, device=f"cuda:{dev}")
            step()
            op_o.gauss_spmv(s_o, s_o, D, h, x_o, y_o)
            torch.cuda.synchronize()
            for _ in range(args.warmup):
                op_o.gauss_spmv(s_o, s_o, D, h, x_o, y_o)
            eo0, eo1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eo0.record(stream)
            for _ in range(args.steps):
                op_o.gauss_spmv(s_o, s_o, D, h, x_o, y_o)
            eo1.record(stream)
            torch.cuda.synchronize()
            yc = y.cpu().numpy()
            yo = y_o.cpu().numpy()[wl.inverse]
            extra_c5["oracle_rows_rel"] = oracle_rows_check(cfg, wl, yc)
            extra_c5 = {**extra_c5, "original_order": {
                "value": nnz_total * args.steps / (eo0.elapsed_time(eo1) * 1e-3),
                "launch_us": eo0.elapsed_time(eo1) * 1e3 / args.steps},
                "cluster_vs_original_rel": float(np.abs(yc - yo).max() / np.abs(yo).max())}
            extra_c5 = {"checks": {k: extra_c5.pop(k) for k in ("oracle_rows_rel", "cluster_vs_original_rel")},
                        **extra_c5}
            del s_o, op_o
            if sched:  # same operator without the schedule: timing + bitwise check
                plain = ShardedOperator(ctx, wl.csr_c, world, rank, layout=layout).op
                y_p = torch.empty_like(y)
                for _ in range(args.warmup):
                    plain.gauss_spmv(s, s, D, h, x, y_p)
                ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ep0.record(stream)
                for _ in range(args.steps):
                    plain.gauss_spmv(s, s, D, h, x, y_p)
                ep1.record(stream)
                torch.cuda.synchronize()
                extra_c5["tree_order_unscheduled"] = {
                    "value": nnz_total * args.steps / (ep0.elapsed_time(ep1) * 1e-3),
                    "launch_us": ep0.elapsed_time(ep1) * 1e3 / args.steps,
                    "bitwise_equal_to_scheduled": bool(torch.equal(y_p, y))}
                plain.close()
            extra_c5["schedule"] = "graph" if sched else "none"
    else:
        y0 = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)  # y_i ~ N(0, 1e-4 I)
        ybuf = [torch.from_numpy(y0[wl.inverse]).to(f"cuda:{dev}"), torch.zeros(n, 2, device=f"cuda:{dev}")]
        f = torch.empty(r1 - r0, 2, device=f"cuda:{dev}")
        ynew = torch.empty(r1 - r0, 2, device=f"cuda:{dev}")
        eta = 4.0 * n / 12.0  # y <- y - eta * F (gradient 4F, learning rate N/12)
        state = {"i": 0}

        def step():
            a, b = ybuf[state["i"] & 1], ybuf[(state["i"] + 1) & 1]
            if world > 1:
                sop.tsne_step(a, 2, f, eta, ynew, b)
            else:
                sop.op.tsne(a, 2, f, False, eta, b)
            state["i"] += 1

        alg = 8 * nnz_local + 4 * (r1 - r0 + 1) + 8 * n + 8 * (r1 - r0) + 8 * (r1 - r0)
        kernel = (f"tsne_group_kernel<G=8{', interleaved, 40 regs' if opts & 2 else ''}> "
                  f"(fused F + y update, {lay_env} layout)")
        work = "t-SNE attractive step with embedding update"

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
    traffic = None  # ncu DRAM bytes of one launch, captured at the full config size on 1 GPU
    tkey = {"c3": "meanshift_lane_kernel", "c4": "tsne_group_kernel_interleaved",
            "c5": "gauss_stream_kernel" if "stream" in kernel else "gauss_warp_kernel"}.get(cfg.name)
    traffic_file = os.path.join(HERE, "profiles", "traffic.json")
    if tkey and world == 1 and os.path.exists(traffic_file):
        with open(traffic_file) as fh:
            traffic = json.load(fh).get(tkey)
    roofline = {"bound": "hbm", "achieved": alg / per / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": alg / per / 1e9 / pk["hbm_gbs"], "traffic": traffic,
                "peak_source": pk["source"], "alg_bytes_per_launch": alg, "kernel": kernel,
                "launch_us": per * 1e6, "basis": "SURVEY.md §8d (per rank)"}
    if cfg.name.startswith("c4") and world == 1:
        # full-size spot check: forces of the first 2048 rows from y0
        from oracle.oracle import Oracle, scale_rel
        y0d = torch.from_numpy(y0[wl.inverse]).to(f"cuda:{dev}")
        f1 = torch.empty(r1 - r0, 2, device=f"cuda:{dev}")
        sop.op.tsne(y0d, 2, f1, False, 0.0, None)
        ctx.sync()
        rp4, cols4, p4 = wl.csr_c.export()
        m4 = 2048
        want = Oracle().tsne_rows(rp4[:m4 + 1], cols4[:int(rp4[m4])], p4[:int(rp4[m4])].astype(np.float64),
                                  y0[wl.inverse].astype(np.float64), m4)
        extra_c5["checks"] = {"oracle_rows_rel": float(scale_rel(f1.cpu().numpy()[:m4], want))}
    if cfg.name.startswith("c3") and world == 1:
        # size-independent check at full size: one step from the initial
        # positions, the first 2048 targets against the double oracle
        out1 = torch.empty_like(s)
        sop.op.meanshift(s, s, D, h, out1)
        ctx.sync()
        extra_c5["checks"] = {"oracle_rows_rel": oracle_rows_check(cfg, wl, out1.cpu().numpy()[:, :D])}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = nonstat_cpu_baseline(cfg, wl, {"c3": 100_000, "c4": 60_000}.get(cfg.name[:2], 4_000))
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "interactions/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": nnz_total * args.steps / (ms * 1e-3), "unit": "interactions/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded mixture, exact device kNN)",
            "config": {"workload": f"{cfg.name}: {work}, N={n}, D={D}, k={cfg.k}, nnz={nnz_total}",
                       "n": n, "dim": D, "k": cfg.k, "nnz": nnz_total,
                       "parallelism": f"row-block x{world}"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": None, "gpu_launches": launches,
            "clocks": clk.summary(), "setup_s": {k: round(v, 2) for k, v in wl.timings.items()},
            **extra_c5,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n", type=int, default=None, help="override the point count (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="c1/c2 at N>1: weak = rank r owns the independent seeded instance "
                         "seed=16r (no data-path collective); strong = one instance, row-block "
                         "sharded with x replicated")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    import torch
    import torch.distributed as dist
    if args.impl == "reference":
        # rank 0 alone times the reference CPU path; no process group, so the
        # idle ranks exit 0 at once instead of waiting in a collective
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if rank == 0:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            run_reference(args, world, rank)
        return
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
                         log=log if rank == 0 else None, seed=16 * rank if weak else 0)
    if args.config in ("c3", "c4", "c5"):
        run_nonstationary(args, cfg, wl, ctx, stream, world, rank, dev)
        if world > 1:
            dist.destroy_process_group()
        return

    # weak: this rank's own instance; strong: its row block of the one
    # cluster-ordered operator (x replicated)
    r0, r1 = shard_rows(cfg.n, world, rank) if not weak else (0, cfg.n)
    csr_local = wl.csr_c.row_block(r0, r1) if (world > 1 and not weak) else wl.csr_c
    op = api.Operator.from_host_csr(ctx, csr_local, api.CLUSTER)
    info = op.info
    x = torch.from_numpy(wl.x_c).to(f"cuda:{dev}")
    y = torch.empty(r1 - r0, dtype=torch.float32, device=f"cuda:{dev}")

    # original-order operator (the spmv_flat path), same rows, for comparison
    op_o = None
    if world == 1:
        op_o = api.Operator.from_host_csr(ctx, wl.csr_o, api.ORIGINAL)
        x_o = torch.from_numpy(wl.x).to(f"cuda:{dev}")
        y_o = torch.empty(cfg.n, dtype=torch.float32, device=f"cuda:{dev}")

    def timed(fn, steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
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

    for _ in range(args.warmup):
        op.spmv(x, y)
    launches0 = ctx.launches
    with ClockSampler(dev) as clk:
        ms = timed(lambda: op.spmv(x, y), args.steps)
    launches = ctx.launches - launches0
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
                "frac": achieved / pk["hbm_gbs"], "traffic": None, "peak_source": pk["source"],
                "alg_bytes_per_launch": ab, "basis": "SURVEY.md §8d CSR basis 8nnz+4(M+1)+4N+4M",
                "format_bytes_per_launch": fb,
                "achieved_format_gbs": fb / per_launch_s / 1e9,
                "frac_format": fb / per_launch_s / 1e9 / pk["hbm_gbs"],
                "kernel": "spmv_tiles_g_kernel<4, pdl>", "launch_us": per_launch_s * 1e6}
    traffic_file = os.path.join(HERE, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            tr = json.load(f).get("spmv_tiles_g_kernel")
        if tr:
            roofline["traffic"] = tr

    extra = {}
    checks = {}
    if world == 1:  # A/B of the cluster-tile kernel variants (K3)
        names = {1: "spmv_tiles_kernel (one CTA per tile, plain loads)",
                 2: "spmv_tiles_bulk_kernel (one CTA per tile, TMA bulk)",
                 5: "spmv_tiles_tma_kernel (persistent, 2-stage TMA ring)",
                 6: "spmv_tiles_g_kernel<8> (unrolled halo stage)",
                 8: "spmv_tiles_g_kernel<4> without programmatic dependent launch",
                 "t64": "default kernel, 64-row tiles",
                 "t256": "default kernel, 256-row tiles"}
        for var in (1, 2, 5, 6, 8, "t64", "t256"):
            tile_rows = 128
            if isinstance(var, str):
                tile_rows = int(var[1:])
            else:
                os.environ["KNNX_SPMV_VARIANT"] = str(var)
            op_v = api.Operator.from_host_csr(ctx, csr_local, api.CLUSTER, tile_rows)
            os.environ.pop("KNNX_SPMV_VARIANT", None)
            y_v = torch.empty_like(y)
            for _ in range(args.warmup):
                op_v.spmv(x, y_v)
            ms_v = timed(lambda: op_v.spmv(x, y_v), args.steps)
            extra[f"cluster_variant_{var}"] = {
                "kernel": names[var], "launch_us": ms_v * 1e3 / args.steps,
                "value": nnz_total * args.steps / (ms_v * 1e-3)}
            checks[f"variant_{var}_rel"] = float(
                (y - y_v).abs().max().item() / max(y_v.abs().max().item(), 1e-30))
            op_v.close()
    if op_o is not None:
        for _ in range(args.warmup):
            op_o.spmv(x_o, y_o)
        ms_o = timed(lambda: op_o.spmv(x_o, y_o), args.steps)
        extra["original_order"] = {
            "value": nnz_total * args.steps / (ms_o * 1e-3), "unit": "interactions/s",
            "launch_us": ms_o * 1e3 / args.steps, "kernel": "spmv_orig_kernel",
            "achieved_gbs": ab / (ms_o * 1e-3 / args.steps) / 1e9}
        # size-independent property: both orders give the same y up to fp32 rounding
        y_c = y.cpu().numpy()
        y_oo = y_o.cpu().numpy()
        checks["cluster_vs_original_rel"] = float(
            np.max(np.abs(y_c[wl.forward] - y_oo)) / np.max(np.abs(y_oo)))

    # end to end through the C ABI with host buffers (H2D x, kernel, D2H y per
    # step), on every rank; whole-job value = all ranks' interactions / the
    # slowest rank's wall time (barrier before each timed call)
    from paper_1709_03671_b200._lib import lib, check
    import ctypes as C
    m_loc = r1 - r0
    xh = torch.from_numpy(wl.x_c).pin_memory()
    yh = torch.empty(m_loc, dtype=torch.float32).pin_memory()
    y_dev = y.cpu().numpy()

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

    def unbatched():
        for _ in range(args.e2e_steps):
            check(lib.knnx_spmv_host(op.h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr())))

    for _ in range(3):
        check(lib.knnx_spmv_host(op.h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr())))
    el = wall_max(unbatched)
    checks["e2e_matches_device"] = bool(np.array_equal(yh.numpy(), y_dev))
    # batched host API: every step still copies its own x in and y out
    xs = torch.from_numpy(np.tile(wl.x_c, (args.e2e_steps, 1))).pin_memory()
    ys = torch.empty(args.e2e_steps, m_loc, dtype=torch.float32).pin_memory()

    def batch():
        check(lib.knnx_spmv_host_batch(op.h, args.e2e_steps, C.c_void_p(xs.data_ptr()),
                                       C.c_void_p(ys.data_ptr())))

    def batch_s():  # median of 3 timed batches (each one API call)
        return sorted(wall_max(batch) for _ in range(3))[1]

    # transfer modes of knnx_spmv_host_batch (runtime.cu): 0 = copy engines
    # both ways, 1 = x by copy engine + the multiply stores y straight into
    # the pinned host buffer, 2 = x by an SM copy from mapped host memory too
    modes = {}
    for mode in (("0", "1", "2", "2:16", "2:64") if world == 1 else ()):
        os.environ["KNNX_E2E_MODE"] = mode.split(":")[0]
        if ":" in mode:
            os.environ["KNNX_E2E_COPY_CTAS"] = mode.split(":")[1]
        ys.zero_()
        check(lib.knnx_spmv_host_batch(op.h, min(3, args.e2e_steps), C.c_void_p(xs.data_ptr()),
                                       C.c_void_p(ys.data_ptr())))
        modes[mode] = nnz_total * args.e2e_steps / batch_s()
        checks[f"e2e_mode{mode}_matches_device"] = bool(
            all(np.array_equal(ys[i].numpy(), y_dev) for i in {0, args.e2e_steps - 1}))
        os.environ.pop("KNNX_E2E_COPY_CTAS", None)
    os.environ.pop("KNNX_E2E_MODE", None)
    check(lib.knnx_spmv_host_batch(op.h, min(3, args.e2e_steps), C.c_void_p(xs.data_ptr()),
                                       C.c_void_p(ys.data_ptr())))
    elb = batch_s()
    checks["e2e_batch_matches_device"] = bool(np.array_equal(ys[-1].numpy(), y_dev))
    rows_total = cfg.n * world if weak else cfg.n
    e2e = {"value": nnz_total * args.e2e_steps / elb, "unit": "interactions/s",
           "h2d_bytes_per_step": 4 * cfg.n * world, "d2h_bytes_per_step": 4 * rows_total,
           "steps": args.e2e_steps,
           "api": "knnx_spmv_host_batch (C ABI, pinned host buffers, default transfer mode)",
           "unbatched_value": nnz_total * args.e2e_steps / el,
           "unbatched_api": "knnx_spmv_host per step"}
    if modes:
        e2e["modes"] = {"ce_both": modes["0"], "ce_in_kernel_out": modes["1"],
                        "sm_in_kernel_out": modes["2"], "sm16_in_kernel_out": modes["2:16"],
                        "sm64_in_kernel_out": modes["2:64"]}

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
            "config": {"workload": f"{cfg.name}: cluster-ordered y=Ax, N={cfg.n}, D={cfg.dim}, "
                                   f"k={cfg.k}, nnz={nnz_total}",
                       "n": cfg.n, "dim": cfg.dim, "k": cfg.k, "nnz": nnz_total,
                       "parallelism": (f"independent instances x{world}" if weak
                                       else f"row-block x{world}"),
                       "tile_rows": info["tile_rows"],
                       "l2": "inputs (188 MB stored) exceed the 126 MB L2; no flush"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "extra": extra, "checks": checks,
            "setup_s": {k: round(v, 2) for k, v in wl.timings.items()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
