"""TEST INFRASTRUCTURE ONLY: the reference arm of bench.py (`--impl reference`).

Builds each BASELINE config's inputs on the CPU without the product library
(libknnx.so is never loaded here) and times the reference's own CPU code path
-- the UNMODIFIED patchord library compiled from /root/reference into
oracle/_ref -- through its public API:

  * points: the oracle's restatement of the workload generators
    (knn_oracle.c orc_gen_*, pinned bitwise to the product's, tests/test_oracle.py);
  * exact kNN: scipy's cKDTree (double precision, every host thread) -- the
    reference's own build_knn (proj/src/knn.cpp:9-62) is O(N^2 D), hours at
    N = 1M; its result is the same exact graph;
  * h = median kNN distance, values by the reference's gaussian_values
    (proj/src/knn.cpp:86-108) with h_ref = h / sqrt(2);
  * ordering: the reference's fit_pca + project + order_tree, i.e.
    make_ordering("tree3") (proj/src/pipeline.cpp:40-45,91-129);
  * the hierarchy: permute + build_hier at the auto cut (proj/src/hier.cpp:40-163);
  * timed: spmv_hier_parallel(hardware_concurrency workers) per step
    (proj/src/kernels.cpp:63-101), the reference's parallel operator.

C3-C5 time the reference's single-threaded non-stationary calls on bounded
samples (meanshift_step, tsne_attractive_step, iterate_interactions).
"""
from __future__ import annotations

import hashlib
import math
import os
import subprocess
import time

import numpy as np

from .oracle import Oracle, Ref, RefHier


def perm_sha(fwd) -> str:
    """sha256 of a forward permutation as little-endian int32 (the key
    tests/golden/perm_hashes.json records)."""
    return hashlib.sha256(np.ascontiguousarray(fwd, "<i4").tobytes()).hexdigest()


def host_cpu(ref: Ref) -> dict:
    """The reference's machine_descriptor() plus lscpu's physical core count."""
    phys = None
    try:
        out = subprocess.run(["lscpu", "-p=core,socket"], capture_output=True, text=True,
                             timeout=10).stdout
        phys = len({ln for ln in out.splitlines() if ln and not ln.startswith("#")})
    except (OSError, subprocess.SubprocessError):
        pass
    return {"machine": ref.machine_descriptor(), "physical_cores": phys,
            "hardware_threads": ref.hardware_threads()}


def knn_cpu(pts64: np.ndarray, k: int, self_set: bool, queries: np.ndarray | None = None):
    """Exact kNN in double precision with scipy's cKDTree over every host
    thread; rows in ascending (distance, index) order like build_knn
    (proj/src/knn.cpp:33-60); self_set drops the query's own point."""
    from scipy.spatial import cKDTree
    q_idx = np.arange(pts64.shape[0]) if queries is None else np.asarray(queries)
    tree = cKDTree(pts64, leafsize=32, balanced_tree=False)
    kk = k + 1 if self_set else k
    d, i = tree.query(pts64[q_idx], k=kk, workers=-1)
    d2 = d * d
    if self_set:
        keep = i != q_idx[:, None]
        # a row keeps its k nearest others (self is normally at position 0)
        order = np.argsort(~keep, axis=1, kind="stable")[:, :k]
        i = np.take_along_axis(i, order, 1)
        d2 = np.take_along_axis(d2, order, 1)
    # ties in distance: ascending index
    o = np.lexsort((i, d2), axis=-1)
    return np.take_along_axis(i, o, 1).astype(np.int32), np.take_along_axis(d2, o, 1)


def median_distance(d2: np.ndarray) -> float:
    return float(np.median(np.sqrt(d2.ravel())))


def c2_workload(n: int = 1_000_000, log=None) -> dict:
    """C2 inputs built entirely by the oracle + the reference (no GPU)."""
    orc, ref = Oracle(), Ref()
    tm = {}
    t0 = time.perf_counter()
    pts = orc.gen_mixture_3level(n, 49, 0.125, 0)
    p64 = pts.astype(np.float64)
    x = orc.gen_uniform01(n, 1).astype(np.float64)
    tm["generate_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ids, d2 = knn_cpu(p64, 30, True)
    tm["knn_s"] = time.perf_counter() - t0
    h = median_distance(d2)
    t0 = time.perf_counter()
    k = ids.shape[1]
    rp = np.arange(0, n * k + 1, k, dtype=np.int64)
    cols = np.sort(ids, axis=1).ravel().astype(np.int32)
    vals = ref.gaussian_values(n, rp, cols, p64, p64, h / math.sqrt(2.0))
    tm["values_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pca = ref.fit_pca(p64, 3)
    tm["order_pca_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    hier, fwd = RefHier.from_original(ref, rp, cols, vals, pca["projected"])
    tm["hier_s"] = time.perf_counter() - t0
    xc = np.empty(n)
    xc[fwd] = x
    if log:
        log(f"[reference c2] n={n} nnz={cols.size} h={h:.4f} pca_iters={pca['iterations']} " +
            " ".join(f"{a}={b:.1f}" for a, b in tm.items()))
    return {"hier": hier, "fwd": fwd, "xc": xc, "nnz": int(cols.size), "h": h, "timings": tm,
            "pca_iterations": pca["iterations"], "ref": ref}


def run_c2(steps: int, warmup: int, n: int = 1_000_000, log=None) -> dict:
    """Time spmv_hier_parallel(all host threads) for `steps` steps after
    `warmup` untimed ones; returns the measurement and its provenance."""
    wl = c2_workload(n, log)
    ref, hier = wl["ref"], wl["hier"]
    hw = ref.hardware_threads()
    hier.bench(wl["xc"], hw, max(1, warmup))
    _, times = hier.bench(wl["xc"], hw, steps)
    times = times.astype(np.float64) * 1e-9
    _, t1 = hier.bench(wl["xc"], 0, 3)
    return {
        "value": wl["nnz"] * steps / float(times.sum()), "ms_per_step": float(times.mean()) * 1e3,
        "median_value": wl["nnz"] / float(np.median(times)), "nnz": wl["nnz"],
        "spmv_hier_1thread": wl["nnz"] / (float(np.median(t1)) * 1e-9),
        "workers": hw, "cut_level": hier.info()["cut_level"],
        "permutation_sha256": perm_sha(wl["fwd"]), "h": wl["h"],
        "pca_iterations": wl["pca_iterations"],
        "setup_s": {a: round(b, 2) for a, b in wl["timings"].items()},
        "host": host_cpu(ref),
    }


def sample_order(ref: Ref, pts64: np.ndarray) -> np.ndarray:
    """The reference's own tree order of a sample (make_ordering("tree3")):
    inverse permutation, i.e. the sample's points in leaf order."""
    fwd, _ = ref.make_ordering("tree3", pts64)
    inv = np.empty_like(fwd)
    inv[fwd] = np.arange(fwd.size, dtype=fwd.dtype)
    return inv


def run_nonstationary(name: str, log=None) -> dict:
    """The reference's single-threaded non-stationary path on a bounded sample
    of C3 / C4 / C5 built without the product: one-call times (median of 3)."""
    orc, ref = Oracle(), Ref()
    if name == "c3":
        n, m = 1_000_000, 100_000
        pts = orc.gen_mixture_3level(n, 49, 0.125, 0).astype(np.float64)
        # sample: 100k targets (seeded), in the reference's tree order of the sample
        rng = np.random.default_rng(0)
        sel = np.sort(rng.choice(n, m, replace=False))
        sel = sel[sample_order(ref, pts[sel])]
        ids, d2 = knn_cpu(pts, 30, False, queries=sel)  # mean-shift rows include self
        h_ref = median_distance(d2) / math.sqrt(2.0)
        uniq, inv = np.unique(ids.ravel(), return_inverse=True)
        times = ref.bench_meanshift(pts[uniq], pts[sel], inv.reshape(m, 30).astype(np.int32),
                                    h_ref, 3) * 1e-9
        nnz = m * 30
        what = (f"meanshift_step on {m} seeded C3 targets in the reference's tree order "
                f"({nnz} interactions, exact cKDTree kNN incl. self)")
    elif name == "c4":
        n, k = 60_000, 90
        pts = orc.gen_mixture_c1(n, 50, 256, 1.0, 0).astype(np.float64)
        pts = pts[sample_order(ref, pts)]
        ids, d2 = knn_cpu(pts, k, True)
        h = median_distance(d2)
        rp = np.arange(0, n * k + 1, k, dtype=np.int64)
        cols = np.sort(ids, axis=1).ravel().astype(np.int32)
        vals = ref.gaussian_values(n, rp, cols, pts, pts, h / math.sqrt(2.0))
        # conditional p_j|i = w / row sum, then P = (P + P^T) / 2n
        vals = vals / np.repeat(np.add.reduceat(vals, rp[:-1]), k)
        r = np.repeat(np.arange(n), k)
        key = np.concatenate([r * n + cols, cols.astype(np.int64) * n + r])
        val = np.concatenate([vals, vals]) / (2.0 * n)
        order = np.argsort(key, kind="stable")
        key, val = key[order], val[order]
        uk, start = np.unique(key, return_index=True)
        pv = np.add.reduceat(val, start)
        srow, scol = (uk // n).astype(np.int32), (uk % n).astype(np.int32)
        srp = np.concatenate([[0], np.cumsum(np.bincount(srow, minlength=n))]).astype(np.int64)
        hier = RefHier.flat(ref, n, n, srp, scol, pv)
        y0 = orc.rng_normal(2, 2 * n).reshape(n, 2) * 1e-2
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            hier.tsne(y0)
            times.append(time.perf_counter() - t0)
        times = np.array(times)
        nnz = int(scol.size)
        what = (f"tsne_attractive_step on a C4-mixture instance of N={n} (k=90 exact kNN, "
                f"symmetrised P, reference tree order; {nnz} entries)")
    elif name == "c5":
        n, m, k = 1_000_000, 4_000, 16
        pts = orc.gen_mixture_aniso(n, 960, 32, 32, 0)
        rng = np.random.default_rng(0)
        sel = np.sort(rng.choice(n, m, replace=False))
        # exact kNN of the sample rows: fp32 screen of the 64 best, exact
        # double re-rank (a tool; the timed call is the reference's)
        p32 = pts
        q = p32[sel]
        qn = (q.astype(np.float64) ** 2).sum(1)
        sn = (p32.astype(np.float64) ** 2).sum(1)
        cand = np.empty((m, 64), np.int64)
        for a in range(0, m, 500):
            g = sn[None, :] - 2.0 * (q[a:a + 500] @ p32.T).astype(np.float64) + qn[a:a + 500, None]
            g[np.arange(g.shape[0]), sel[a:a + 500]] = np.inf
            cand[a:a + 500] = np.argpartition(g, 64, axis=1)[:, :64]
        d2 = ((pts[cand].astype(np.float64) - q[:, None, :].astype(np.float64)) ** 2).sum(-1)
        o = np.argsort(d2, axis=1, kind="stable")[:, :k]
        ids = np.take_along_axis(cand, o, 1)
        h_ref = median_distance(np.take_along_axis(d2, o, 1)) / math.sqrt(2.0)
        uniq, inv = np.unique(ids.ravel(), return_inverse=True)
        rp = np.arange(0, m * k + 1, k, dtype=np.int64)
        hier = RefHier.flat(ref, m, uniq.size, rp, inv.astype(np.int32), np.ones(m * k))
        xs = np.tile(orc.gen_uniform01(n, 1)[uniq].astype(np.float64), (3, 1))
        _, t_ns = hier.iterate_gaussian(q.astype(np.float64), pts[uniq].astype(np.float64), h_ref, xs)
        times = t_ns * 1e-9
        nnz = m * k
        what = (f"iterate_interactions (Gaussian update_values + spmv_hier) for {m} seeded C5 "
                f"rows ({nnz} interactions, D=960)")
    else:
        raise ValueError(name)
    med = float(np.median(times))
    if log:
        log(f"[reference {name}] {what}: {nnz / med:.3e} interactions/s")
    return {"value": nnz / med, "ms_per_step": med * 1e3, "sample": what,
            "host": host_cpu(ref)}
