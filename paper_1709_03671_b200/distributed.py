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


class RowGather:
    """All-gather of row blocks into a full (n_rows x ...) tensor with
    persistent buffers: each rank's block is padded to max_rows (blocks are
    tile-aligned, so they differ by at most one granule), gathered with one
    all_gather_into_tensor, and the padded stack is compacted by one device
    gather (knnx_gather_rows_dev) through a precomputed index -- no per-call
    allocation, one collective and one kernel per exchange."""

    def __init__(self, shard: Shard, tail: tuple, dtype, device, ctx=None, group=None):
        import torch
        self.shard, self.group, self.ctx = shard, group, ctx
        self.pad = torch.zeros((shard.max_rows,) + tuple(tail), dtype=dtype, device=device)
        self.stack = torch.empty((shard.world * shard.max_rows,) + tuple(tail), dtype=dtype,
                                 device=device)
        idx = np.concatenate([np.arange(a, b) - a + r * shard.max_rows
                              for r, (a, b) in enumerate(shard.blocks)]).astype(np.int32)
        self.index = torch.from_numpy(idx).to(device) if str(device) != "cpu" else torch.from_numpy(idx)
        self.equal = all(b - a == shard.max_rows for a, b in shard.blocks)

    def __call__(self, local, out):
        import torch
        import torch.distributed as dist
        shard = self.shard
        if shard.world > 1 and dist.get_backend(self.group) == "nccl":
            if self.equal:  # blocks of one size: gather straight into out
                dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)
                return out
            self.pad[: local.shape[0]] = local
            dist.all_gather_into_tensor(self.stack, self.pad, group=self.group)
        elif shard.world > 1:  # gloo (CPU tests): list form
            self.pad[: local.shape[0]] = local
            dist.all_gather(list(self.stack.chunk(shard.world)), self.pad, group=self.group)
        else:
            out[: local.shape[0]] = local
            return out
        if self.ctx is not None and out.is_cuda:
            self.ctx.gather_rows(self.stack, self.index, out)
        else:
            out.copy_(self.stack.index_select(0, self.index.to(self.stack.device).long()))
        return out


def all_gather_rows(local, shard: Shard, out, group=None, ctx=None):
    """One-shot form of RowGather (allocates its buffers; the iterating
    helpers below keep a RowGather instead)."""
    return RowGather(shard, tuple(local.shape[1:]), local.dtype, local.device, ctx, group)(local, out)


def join_library_stream(ctx) -> None:
    """Make torch's current stream wait for the library's stream, so torch /
    NCCL work issued next sees results the library launched on its own
    (non-blocking) stream."""
    import torch
    from ._lib import lib
    handle = lib.knnx_ctx_stream(ctx.h)
    cur = torch.cuda.current_stream()
    if handle and int(handle) != int(cur.cuda_stream):
        cur.wait_stream(torch.cuda.ExternalStream(int(handle), device=cur.device))


class ShardedOperator:
    """This rank's row block of a cluster-ordered operator on its GPU."""

    def __init__(self, ctx, csr, world: int, rank: int, tile_rows: int = 256, group=None,
                 layout=None, schedule: bool = False, options: int = 0, dev_csr=None):
        """layout: api.CLUSTER (16-bit halo tiles, default) or api.ORIGINAL
        (int32 columns on the same tree-ordered rows: fewer dependent loads
        for high-degree graphs whose tile halos are large).  schedule: run
        the shard's rows in the graph-locality schedule (KNNX_SCHEDULE_GRAPH;
        results unchanged).  dev_csr: the same matrix as an api.DeviceCsr; a
        single-rank original-layout scheduled operator is then built on the
        device."""
        from . import api
        row_ptr, _, _ = csr.export()
        self.shard = Shard(world, rank, partition_rows(row_ptr, world, tile_rows))
        self.group = group
        block = csr.row_block(self.shard.r0, self.shard.r1) if world > 1 else csr
        lay = api.CLUSTER if layout is None else layout
        if (dev_csr is not None and schedule and lay == api.ORIGINAL and tile_rows == 256
                and (options & ~api.OPT_GROUP_INTERLEAVE) == 0):
            # the whole operator (schedule, tile sort, placement) is built on
            # the device from the CSR already there (knnx_op_create_csr_dev);
            # a rank of several takes its row block of the full matrix
            r0, r1 = self.shard.r0, self.shard.r1
            self.op = api.Operator.from_csr_device(
                ctx, 0, 0, dev_csr, schedule="graph", options=options, col_base=r0,
                rows=None if world == 1 else (r0, r1),
                block_nnz=int(row_ptr[r1] - row_ptr[r0]))
        elif schedule:
            m, n, _nnz, _ = block.shape
            rp, cols, vals = block.export()
            self.op = api.Operator.from_csr_scheduled(ctx, m, n, rp, cols, vals, lay, tile_rows,
                                                      None, self.shard.r0, options)
        else:
            self.op = api.Operator.from_host_csr(ctx, block, lay, tile_rows)
        self.op.set_row_base(self.shard.r0)
        self.ctx = ctx
        self._gathers: dict = {}

    def _gather(self, local, out):
        key = (tuple(local.shape[1:]), local.dtype, str(local.device))
        g = self._gathers.get(key)
        if g is None:
            g = self._gathers[key] = RowGather(self.shard, key[0], local.dtype, local.device,
                                               self.ctx, self.group)
        return g(local, out)

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
        join_library_stream(self.ctx)
        m = y_local.abs().max().reshape(1) if y_local.numel() else torch.zeros(1, device=y_local.device)
        if self.shard.world > 1:
            dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
        self._gather(y_local, x_next_full)
        x_next_full /= m
        return x_next_full

    def meanshift_step(self, t_full, s_full, dim: int, h: float, t_local_out, t_full_out=None):
        """New positions of this rank's targets; optionally all-gathered."""
        r0, r1 = self.rows
        self.op.meanshift(t_full[r0:r1], s_full, dim, h, t_local_out)
        if t_full_out is not None:
            join_library_stream(self.ctx)
            self._gather(t_local_out, t_full_out)
        return t_local_out

    def enable_fused_tsne(self, y_bufs) -> None:
        """Fused t-SNE exchange (multi-process, one GPU per rank): every
        rank maps every other rank's replicated embedding buffers (CUDA IPC,
        knnx_ipc_*), so the force kernel stores its updated rows straight
        into all replicas over NVLink (knnx_tsne_attr_peers_dev) and a
        stream-ordered NCCL barrier (knnx_comm_barrier) replaces the
        all-gather after the kernel.  y_bufs: this rank's full-size embedding
        buffers (e.g. the double buffer of the iteration)."""
        import ctypes as C

        import torch.distributed as dist

        from . import api
        from ._lib import check, lib
        world, rank = self.shard.world, self.shard.rank
        uid = [api.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0, group=self.group)
        self.comm = api.Comm(self.ctx, world, rank, uid[0])
        self._ipc_open = []
        self.fused_outs = []
        for buf in y_bufs:
            h = C.create_string_buffer(64)
            check(lib.knnx_ipc_get_handle(self.ctx.h, C.c_void_p(buf.data_ptr()), h))
            handles = [None] * world
            dist.all_gather_object(handles, h.raw, group=self.group)
            ptrs = []
            for q, hq in enumerate(handles):
                if q == rank:
                    ptrs.append(buf.data_ptr())
                    continue
                p = C.c_void_p()
                check(lib.knnx_ipc_open(self.ctx.h, C.create_string_buffer(hq, 64), C.byref(p)))
                self._ipc_open.append(p)
                ptrs.append(p.value)
            self.fused_outs.append(ptrs)

    def tsne_step_fused(self, y_full, dim: int, f_local, step: float, out_index: int):
        """Forces of this rank's rows; y - step F stored into buffer
        `out_index` (of enable_fused_tsne) on every rank; then the barrier."""
        self.op.tsne_peers(y_full, dim, f_local, step, self.fused_outs[out_index])
        self.comm.barrier()

    def tsne_step(self, y_full, dim: int, f_local, step: float, y_local_out, y_full_out):
        """Forces on this rank's points, y update, embedding all-gather."""
        self.op.tsne(y_full, dim, f_local, False, step, y_local_out)
        join_library_stream(self.ctx)
        self._gather(y_local_out, y_full_out)
        return y_full_out
