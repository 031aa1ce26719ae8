"""Row-block sharding of a cluster-ordered operator across GPUs.

One process per GPU (torch.distributed, NCCL over NVLink for the data plane,
gloo on CPU for the tests).  The cluster-ordered rows are cut into contiguous
blocks on tile boundaries, balanced by nonzeros; each rank owns its block's
operator and its rows of every per-target array.  Each row's accumulation
stays on one GPU, so sharded results are bit-identical to one GPU.

Exchanges (each only where the algorithm has one):
  * stationary y = A x with fixed x: none;
  * power iteration x <- y / max|y| (C2 variant): all-gather of y (4 B/row)
    plus one max all-reduce per iteration;
  * mean shift (C3): all-gather of the moved targets (4 D B/row) -- the
    BASELINE-mandated coordinate exchange; nothing in the next step waits on
    it when sources are fixed, so it runs on a side stream;
  * t-SNE (C4): all-gather of the 2-D embedding every iteration (8 B/row).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition_rows(row_ptr: np.ndarray, world: int, granule: int = 128) -> list[tuple[int, int]]:
    """Contiguous row blocks cut on `granule` boundaries with ~equal nonzeros."""
    row_ptr = np.asarray(row_ptr, np.int64)
    n = row_ptr.size - 1
    n_gran = (n + granule - 1) // granule
    cuts_rows = np.minimum(np.arange(n_gran + 1) * granule, n)
    cum = row_ptr[cuts_rows]  # nonzeros before each granule boundary
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        g = int(np.searchsorted(cum, target))
        if g > 0 and g <= n_gran and target - cum[g - 1] < cum[min(g, n_gran)] - target:
            g -= 1  # the nearer granule boundary
        g = min(max(g, bounds[-1]), n_gran)
        bounds.append(g)
    bounds.append(n_gran)
    return [(int(cuts_rows[bounds[i]]), int(cuts_rows[bounds[i + 1]])) for i in range(world)]


@dataclass
class Shard:
    world: int
    rank: int
    blocks: list[tuple[int, int]]

    @property
    def r0(self) -> int:
        return self.blocks[self.rank][0]

    @property
    def r1(self) -> int:
        return self.blocks[self.rank][1]

    @property
    def max_rows(self) -> int:
        return max(b - a for a, b in self.blocks)

    @property
    def n_rows(self) -> int:
        return self.blocks[-1][1]


def all_gather_rows(local, shard: Shard, out, group=None):
    """Gather every rank's row block of a (rows x ...) tensor into `out`
    (n_rows x ...).  Blocks may differ in length: each rank contributes a
    max_rows-padded chunk through all_gather_into_tensor, then the padded
    stack is compacted on the device."""
    import torch
    import torch.distributed as dist
    tail = tuple(local.shape[1:])
    pad = torch.zeros((shard.max_rows,) + tail, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    stack = torch.empty((shard.world * shard.max_rows,) + tail, dtype=local.dtype,
                        device=local.device)
    if shard.world > 1 and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(stack, pad, group=group)
    elif shard.world > 1:  # gloo (CPU tests): list form
        dist.all_gather(list(stack.chunk(shard.world)), pad, group=group)
    else:
        stack.copy_(pad)
    for r, (a, b) in enumerate(shard.blocks):
        out[a:b] = stack[r * shard.max_rows: r * shard.max_rows + (b - a)]
    return out


class ShardedOperator:
    """This rank's row block of a cluster-ordered operator on its GPU."""

    def __init__(self, ctx, csr, world: int, rank: int, tile_rows: int = 256, group=None,
                 layout=None, schedule: bool = False, options: int = 0):
        """layout: api.CLUSTER (16-bit halo tiles, default) or api.ORIGINAL
        (int32 columns on the same tree-ordered rows: fewer dependent loads
        for high-degree graphs whose tile halos are large).  schedule: run
        the shard's rows in the graph-locality schedule (KNNX_SCHEDULE_GRAPH;
        results unchanged)."""
        from . import api
        row_ptr, _, _ = csr.export()
        self.shard = Shard(world, rank, partition_rows(row_ptr, world, tile_rows))
        self.group = group
        block = csr.row_block(self.shard.r0, self.shard.r1) if world > 1 else csr
        lay = api.CLUSTER if layout is None else layout
        if schedule:
            m, n, _nnz, _ = block.shape
            rp, cols, vals = block.export()
            self.op = api.Operator.from_csr_scheduled(ctx, m, n, rp, cols, vals, lay, tile_rows,
                                                      None, self.shard.r0, options)
        else:
            self.op = api.Operator.from_host_csr(ctx, block, lay, tile_rows)
        self.op.set_row_base(self.shard.r0)
        self.ctx = ctx

    @property
    def rows(self) -> tuple[int, int]:
        return self.shard.r0, self.shard.r1

    def spmv(self, x_full, y_local) -> None:
        self.op.spmv(x_full, y_local)

    def power_step(self, x_full, y_local, x_next_full):
        """x_next = y / max|y| over all ranks (one max all-reduce + all-gather)."""
        import torch
        import torch.distributed as dist
        self.op.spmv(x_full, y_local)
        m = y_local.abs().max().reshape(1) if y_local.numel() else torch.zeros(1, device=y_local.device)
        if self.shard.world > 1:
            dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
        all_gather_rows(y_local, self.shard, x_next_full, self.group)
        x_next_full /= m
        return x_next_full

    def meanshift_step(self, t_full, s_full, dim: int, h: float, t_local_out, t_full_out=None):
        """New positions of this rank's targets; optionally all-gathered."""
        r0, r1 = self.rows
        self.op.meanshift(t_full[r0:r1], s_full, dim, h, t_local_out)
        if t_full_out is not None:
            all_gather_rows(t_local_out, self.shard, t_full_out, self.group)
        return t_local_out

    def tsne_step(self, y_full, dim: int, f_local, step: float, y_local_out, y_full_out):
        """Forces on this rank's points, y update, embedding all-gather."""
        self.op.tsne(y_full, dim, f_local, False, step, y_local_out)
        all_gather_rows(y_local_out, self.shard, y_full_out, self.group)
        return y_full_out
