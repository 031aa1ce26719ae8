"""Seeded synthetic workloads for the BASELINE.json configs.

Every config is generated deterministically from Rng (mt19937_64, the
reference's generator) and then built with the framework's own tools:
bit-exact tree ordering (host C++, PCA covariance on the device), the exact
device kNN in cluster order, Gaussian values by the operator's own
update_values path.  BASELINE's weight convention exp(-d^2/h^2) with h the
median kNN distance is expressed through the reference convention
exp(-d^2/(2 h_ref^2)) with h_ref = h / sqrt(2).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import api

# sub-seed derivation: Rng(seed + stream_id)
SEED_POINTS, SEED_CHARGE, SEED_EMBED = 0, 1, 2


@dataclass
class Config:
    name: str
    n: int
    dim: int
    k: int
    kind: int
    n_clusters: int = 0
    p0: float = 1.0
    self_in_knn: bool = False   # mean-shift semantics: targets' own point included
    symmetrize: bool = False
    iterations: int = 10


CONFIGS = {
    # C1: 64-component mixture, means U[-10,10]^49, sigma 1, k=30
    "c1": Config("c1", 20_000, 49, 30, api.GEN_C1_MIXTURE, 64, 1.0, iterations=10),
    # C2: 3-level mixture 16x16x16, scales 10/2/0.5, point noise 0.125, k=30
    "c2": Config("c2", 1_000_000, 49, 30, api.GEN_3LEVEL, 0, 0.125, iterations=100),
    # C3: same points, mean-shift neighbor lists (self included), 20 steps
    "c3": Config("c3", 1_000_000, 49, 30, api.GEN_3LEVEL, 0, 0.125, self_in_knn=True,
                 iterations=20),
    # C4: 4M x 50, 256-component mixture (means U[-10,10], sigma 1), k=90 symmetrised
    "c4": Config("c4", 4_000_000, 50, 90, api.GEN_C1_MIXTURE, 256, 1.0, symmetrize=True,
                 iterations=50),
    # C5: 1M x 960, 32 x 32 anisotropic clusters, k=16
    "c5": Config("c5", 1_000_000, 960, 16, api.GEN_ANISO, (32 << 16) | 32, 1.0, iterations=20),
}


def scaled(name: str, n: int) -> Config:
    c = CONFIGS[name]
    return Config(c.name + f"@{n}", n, c.dim, c.k, c.kind, c.n_clusters, c.p0, c.self_in_knn,
                  c.symmetrize, c.iterations)


@dataclass
class Workload:
    cfg: Config
    points: np.ndarray            # n x dim fp32, original (generation) order
    forward: np.ndarray           # tree leaf order: forward[original] = cluster position
    inverse: np.ndarray
    tree: api.Tree
    embedding: np.ndarray         # n x 3 PCA projection the tree was built on
    knn_ids_c: np.ndarray         # cluster order neighbor ids (cluster positions), n x k
    knn_d2_c: np.ndarray
    h_baseline: float             # median kNN distance (BASELINE convention)
    csr_c: api.HostCsr            # cluster order, Gaussian values
    x: np.ndarray                 # charge U[0,1], original order
    timings: dict = field(default_factory=dict)
    _csr_o: Optional[api.HostCsr] = None
    dev_csr: Optional[object] = None   # api.DeviceCsr of csr_c when build(keep_device_csr=True)

    @property
    def csr_o(self) -> api.HostCsr:
        """Original order, same values: permuted on first use (a host sort of
        every entry, ~1 min at C4's 6e8 entries, which the C3/C4 benches never
        read)."""
        if self._csr_o is None:
            self._csr_o = self.csr_c.permute(self.inverse)
        return self._csr_o

    @property
    def h_ref(self) -> float:
        return self.h_baseline / math.sqrt(2.0)

    @property
    def points_c(self) -> np.ndarray:
        out = np.empty_like(self.points)
        out[self.forward] = self.points
        return out

    @property
    def x_c(self) -> np.ndarray:
        out = np.empty_like(self.x)
        out[self.forward] = self.x
        return out

    @property
    def nnz(self) -> int:
        return self.csr_c.shape[2]


def build(cfg: Config, ctx: api.Context, device: int = 0, with_values: bool = True,
          log=None, seed: int = 0, pca_device: Optional[int] = None,
          knn_impl: str = "auto", keep_device_csr: bool = False) -> Workload:
    """Generate one seeded instance of `cfg`.  `seed` offsets every sub-stream
    (Rng(seed + stream_id)); bench.py's weak-scaling mode gives rank r the
    independent instance seed = 16 r (rank 0 is the single-GPU workload).
    pca_device: device for the PCA covariance action (default `device`;
    -1 = the host loop, bitwise the same result).  knn_impl: "auto" (the exact
    SIMT search for dim <= 64 and k <= 32, the tensor-core screen + exact
    re-rank otherwise), "simt" or "tensor"."""
    import torch

    tm = {}
    t0 = time.perf_counter()
    pts = api.gen_points(cfg.kind, cfg.n, cfg.dim, cfg.n_clusters, cfg.p0, seed + SEED_POINTS)
    tm["generate_s"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    pts64 = pts.astype(np.float64)
    pca = api.fit_pca(pts64, 3, pca_device=device if pca_device is None else pca_device)
    # the tree over the projection: on the device when the PCA ran there
    # (two sorts over the orthant paths, the same tree as the host recursion)
    pdev = device if pca_device is None else pca_device
    tree = api.build_tree(pca["projected"], 128, 12, device=pdev)
    tree.pca_iterations = pca["iterations"]
    tm["order_s"] = time.perf_counter() - t0
    fwd = tree.forward
    inv = np.empty_like(fwd)
    inv[fwd] = np.arange(cfg.n, dtype=np.int32)

    t0 = time.perf_counter()
    # cluster-ordered points on the device: upload in generation order and
    # apply the permutation there (K1), instead of permuting 3.8 GB on the host
    src = api.to_device_points(pts, f"cuda:{device}")
    dev_pts = torch.empty_like(src)
    ctx.permute_rows(src, torch.from_numpy(fwd).to(f"cuda:{device}"), dev_pts)
    ctx.sync()
    del src
    if cfg.dim <= 64 and cfg.k <= 32 and knn_impl != "tensor":
        # provably exact block-pruned search (knnx_knn_dev)
        ids, d2 = ctx.knn(dev_pts, dev_pts, cfg.n, cfg.n, cfg.dim, cfg.k, self_set=not cfg.self_in_knn)
        ctx.sync()
    elif knn_impl == "simt":
        ids, d2 = ctx.knn(dev_pts, dev_pts, cfg.n, cfg.n, cfg.dim, cfg.k, self_set=not cfg.self_in_knn)
        ctx.sync()
    else:
        # wide rows (C5, D = 960) and long lists (C4, k = 90): the tcgen05
        # distance screen + exact fp32 re-rank (knnx_knn_wide_dev); the margin
        # statistics go to the timings
        ids, d2, knn_stats = ctx.knn_wide(dev_pts, dev_pts, cfg.n, cfg.n, cfg.dim, cfg.k,
                                          self_set=not cfg.self_in_knn, want_stats=True)
        ctx.sync()
        tm["knn_wide"] = knn_stats
    torch.cuda.synchronize(device)
    tm["knn_s"] = time.perf_counter() - t0
    ids_c = ids.cpu().numpy()
    d2_c = d2.cpu().numpy()
    h = api.median_distance(d2_c)

    t0 = time.perf_counter()
    dev_csr = None
    if cfg.symmetrize:
        # t-SNE joint affinities (C4), built on the device from the kNN rows:
        # p_j|i = exp(-d^2/h^2) / row sum, P = (P_cond + P_cond^T) / 2N
        # (knnx_tsne_affinities_dev; sums to 1)
        res = ctx.tsne_affinities(ids, d2, h / math.sqrt(2.0), 1.0 / (2.0 * cfg.n),
                                  keep_device=keep_device_csr)
        rp, cols, vals = res[:3]
        dev_csr = res[3] if keep_device_csr else None
        csr_c = api.HostCsr.from_arrays(cfg.n, cfg.n, rp, cols, vals)
        with_values = False
    else:
        csr_c = api.HostCsr.from_knn(ids_c, cfg.n)
    if with_values:
        if cfg.k <= 32:  # tiles built on the device straight from the kNN rows
            op = api.Operator.from_knn_device(ctx, ids, cfg.n)
        else:
            m, n, _nnz, _ = csr_c.shape
            rp, cols, _ = csr_c.export()
            op = api.Operator.from_csr(ctx, m, n, rp, cols, None, api.CLUSTER)
        op.update_gaussian(dev_pts, dev_pts, cfg.dim, h / math.sqrt(2.0))
        ctx.sync()
        csr_c.set_values(op.get_values())
        op.close()
    tm["format_s"] = time.perf_counter() - t0
    del dev_pts
    x = api.gen_uniform01(cfg.n, seed + SEED_CHARGE)
    if log:
        log(f"[workload {cfg.name}] n={cfg.n} dim={cfg.dim} k={cfg.k} nnz={csr_c.shape[2]} "
            f"h={h:.4f} pca_iters={pca['iterations']} " +
            " ".join(f"{k}={v:.2f}" if isinstance(v, float) else f"{k}={v}" for k, v in tm.items()))
    wl = Workload(cfg, pts, fwd, inv, tree, pca["projected"], ids_c, d2_c, h, csr_c, x, tm)
    wl.dev_csr = dev_csr
    return wl
