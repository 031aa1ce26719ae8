"""Generate tests/golden/golden_small.npz by running the REFERENCE LIBRARY ITSELF
(oracle/_ref/libpatchord_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run here, where the reference tree exists:

    make -C oracle && python tests/golden/make_golden.py

The fixture pins the CPU oracle restatement (tests/test_golden.py) and the
GPU kernels (tests/test_gpu_golden.py) on the GPU box, where /root/reference
does not exist.  Every array below is an output of the reference's own code.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref, RefHier, _p  # noqa: E402


def main():
    ref = Ref()
    out = {}
    for seed in (0, 1, 42):
        out[f"rng_u64_{seed}"] = ref.rng_u64(seed, 64)
        out[f"rng_uniform01_{seed}"] = ref.rng_uniform01(seed, 64)
        out[f"rng_normal_{seed}"] = ref.rng_normal(seed, 65)
        out[f"order_scattered_{seed}"] = ref.order_scattered(300, seed)

    # reference generator: 8-component mixture (proj/src/synth.cpp:60-74)
    n, dim, k = 512, 6, 8
    pts = np.empty((n, dim))
    ref._ok(ref.lib.ref_gen_gaussian_mixture(n, dim, 8, 40.0, 1.5, 21, _p(pts)))
    pts = pts.astype(np.float32).astype(np.float64)  # fp32-representable inputs
    out["points"] = pts
    ids, d2 = ref.build_knn(pts, None, k, True)
    out["knn_ids"], out["knn_d2"] = ids, d2
    for scheme in ("tree2", "tree3"):
        out[f"forward_{scheme}"], out[f"ratio_{scheme}"] = ref.make_ordering(scheme, pts)
    pca = ref.fit_pca(pts, 3)
    out["pca_axes"], out["pca_projected"] = pca["axes"], pca["projected"]
    out["pca_iterations"] = np.int64(pca["iterations"])

    # canonical pattern + Gaussian values (knn.cpp:86-108), h = 2.0
    cols = np.sort(ids, axis=1).ravel().astype(np.int32)
    rows = np.repeat(np.arange(n, dtype=np.int32), k)
    rp = np.arange(n + 1, dtype=np.int64) * k
    h = 2.0
    vals = np.empty(cols.size)
    ref._ok(ref.lib.ref_gaussian_values(n, n, cols.size, _p(rows), _p(cols), _p(pts), _p(pts), dim, h,
                                        _p(vals)))
    out["row_ptr"], out["cols"], out["vals"], out["h"] = rp, cols, vals, np.float64(h)
    # every input the GPU sees is fp32: round charges, targets, affinities and
    # the embedding to fp32 before the reference runs
    f32 = lambda a: np.asarray(a).astype(np.float32).astype(np.float64)  # noqa: E731
    x = f32(ref.rng_uniform01(5, n))
    out["x"] = x
    out["y_flat"] = ref.spmv_flat(n, rp, cols, vals, x)

    # cluster order: the reference's own tree, permute and blocked operator
    hier, fwd = RefHier.from_original(ref, rp, cols, vals, pca["projected"], 32, 12, -1)
    r, c, v = hier.flatten()
    out["hier_forward"], out["hier_rows"], out["hier_cols"], out["hier_vals"] = fwd, r, c, v
    xc = np.empty(n)
    xc[fwd] = x
    out["x_cluster"] = xc
    out["y_hier"] = hier.spmv(xc)
    out["hier_cut_level"] = np.int64(hier.info()["cut_level"])
    hier.dump(os.path.join(HERE, "golden_small.hbm1"))  # the reference's own HBM1 writer

    # iterate_interactions with the Gaussian value model, 2 steps
    xs = f32(np.stack([ref.rng_uniform01(6, n), ref.rng_uniform01(7, n)]))
    pc = ref.permute_points(pts, fwd)
    out["points_cluster"] = pc
    out["iterate_xs"] = xs
    out["iterate_ys"], _ = hier.iterate_gaussian(pc, pc, h, xs)

    # mean-shift step over the reference's kNN rows (self excluded here)
    t = f32(pts + 0.25)
    out["ms_targets"] = t
    out["ms_out"] = ref.meanshift_step(pts, t, ids, h)

    # t-SNE attractive step on a symmetrised pattern (build_hier_flat, n <= 65536)
    sr, sc = ref.symmetrize(rp, cols)
    srp = np.zeros(n + 1, np.int64)
    np.add.at(srp, sr + 1, 1)
    srp = np.cumsum(srp)
    p = ref.rng_uniform01(8, sc.size) + 0.1
    p = f32(p / p.sum())
    y2 = f32(ref.rng_normal(9, 2 * n).reshape(n, 2) * 1e-2)
    flat = RefHier.flat(ref, n, n, srp, sc, p)
    out["tsne_row_ptr"], out["tsne_cols"], out["tsne_p"], out["tsne_y"] = srp, sc, p, y2
    out["tsne_f"] = flat.tsne(y2)
    out["tsne_a"] = flat.flatten()[2]

    path = os.path.join(HERE, "golden_small.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
