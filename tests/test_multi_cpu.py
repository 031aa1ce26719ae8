"""Multi-rank path on CPU: world_size 2 over gloo (no GPU).

The per-rank compute is the CPU oracle standing in for the kernels (this is a
test, so it may call the checker); what is under test is the product's
distribution logic -- nnz-balanced tile-aligned row blocks (partition_rows),
the row-block shards (HostCsr.row_block), and the padded all-gather
(all_gather_rows) -- and that sharded results are bit-identical to the
unsharded ones, as SURVEY.md §8e requires (each row's sum stays on one rank).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1709_03671_b200.distributed import Shard, all_gather_rows, partition_rows

G = os.path.join(os.path.dirname(__file__), "golden", "golden_small.npz")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_1709_03671_b200 import api
        orc = Oracle()
        g = np.load(G)
        n = g["x"].size
        rp, cols, vals = g["row_ptr"], g["cols"], g["vals"]
        csr = api.HostCsr.from_arrays(n, n, rp, cols, vals.astype(np.float32))
        shard = Shard(world, rank, partition_rows(rp, world, granule=32))
        blk_rp, blk_cols, blk_vals = csr.row_block(shard.r0, shard.r1).export()

        # stationary y = A x: no exchange; gather only to compare
        y_loc = orc.spmv(blk_rp, blk_cols, blk_vals.astype(np.float64), g["x"])
        y_full = torch.zeros(n, dtype=torch.float64)
        all_gather_rows(torch.from_numpy(y_loc), shard, y_full)

        # power iteration x <- y / max|y|: max all-reduce + all-gather of y
        x = torch.from_numpy(g["x"].copy())
        for _ in range(3):
            yl = torch.from_numpy(orc.spmv(blk_rp, blk_cols, blk_vals.astype(np.float64), x.numpy()))
            m = yl.abs().max().reshape(1)
            dist.all_reduce(m, op=dist.ReduceOp.MAX)
            nxt = torch.zeros(n, dtype=torch.float64)
            all_gather_rows(yl, shard, nxt)
            x = nxt / m

        # mean shift with the coordinate all-gather of the moved targets
        k = g["knn_ids"].shape[1]
        ids = g["knn_ids"]
        t = torch.from_numpy(g["ms_targets"].copy())
        for _ in range(3):
            tl = orc.meanshift_step(ids[shard.r0:shard.r1], t.numpy()[shard.r0:shard.r1],
                                    g["points"], float(g["h"]))
            nt = torch.zeros_like(t)
            all_gather_rows(torch.from_numpy(tl), shard, nt)
            t = nt

        # t-SNE direct forces on a row block + embedding all-gather
        srp, scol, p = g["tsne_row_ptr"], g["tsne_cols"], g["tsne_p"]
        tsh = Shard(world, rank, partition_rows(srp, world, granule=32))
        y = torch.from_numpy(g["tsne_y"].copy())
        for _ in range(2):
            a, b = tsh.r0, tsh.r1
            lrp = srp[a:b + 1] - srp[a]
            f = np.zeros((b - a, 2))
            for i in range(b - a):
                for e in range(lrp[i], lrp[i + 1]):
                    j = scol[srp[a] + e]
                    d = y[a + i].numpy() - y[j].numpy()
                    f[i] += p[srp[a] + e] / (1.0 + d @ d) * d
            ny = torch.zeros_like(y)
            all_gather_rows(y[a:b] - 100.0 * torch.from_numpy(f), tsh, ny)
            y = ny
        if rank == 0:
            results["y"] = y_full.numpy()
            results["x"] = x.numpy()
            results["t"] = t.numpy()
            results["emb"] = y.numpy()
            results["blocks"] = shard.blocks
            results["k"] = k
    finally:
        dist.destroy_process_group()


def test_partition_rows_balances_nnz():
    rp = np.concatenate([[0], np.cumsum(np.r_[np.full(500, 10), np.full(524, 40)])])
    for world in (1, 2, 3, 4, 8):
        blocks = partition_rows(rp, world, granule=32)
        assert blocks[0][0] == 0 and blocks[-1][1] == 1024
        assert all(a == blocks[i - 1][1] for i, (a, _) in enumerate(blocks) if i)
        assert all(a % 32 == 0 for a, _ in blocks)
        nnz = [rp[b] - rp[a] for a, b in blocks]
        assert max(nnz) - min(nnz) <= 2 * 32 * 40  # each cut within half a granule


def test_two_ranks_gloo_bit_identical(oracle):
    g = np.load(G)
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
        res = dict(results)
    n = g["x"].size
    # unsharded references
    v32 = g["vals"].astype(np.float32).astype(np.float64)  # the shards hold fp32 values
    y = oracle.spmv(g["row_ptr"], g["cols"], v32, g["x"])
    assert np.array_equal(res["y"], y)
    x = g["x"].copy()
    for _ in range(3):
        yy = oracle.spmv(g["row_ptr"], g["cols"], v32, x)
        x = yy / np.abs(yy).max()
    assert np.array_equal(res["x"], x)
    t = g["ms_targets"].copy()
    for _ in range(3):
        t = oracle.meanshift_step(g["knn_ids"], t, g["points"], float(g["h"]))
    assert np.array_equal(res["t"], t)
    assert len(res["blocks"]) == 2 and res["blocks"][1][1] == n
