"""C-ABI behaviour on the GPU: batched host/device entry points, validation
errors with the reference's errc names, stream handling."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import scale_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small(ctx):
    from paper_1709_03671_b200 import workloads
    return workloads.build(workloads.scaled("c1", 2000), ctx, 0)


def test_host_batch_and_graph_batch(ctx, small, oracle):
    import torch

    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import check, lib
    rp, cols, vals = small.csr_c.export()
    n = small.cfg.n
    op = api.Operator.from_csr(ctx, n, n, rp, cols, vals, api.CLUSTER)
    rng = np.random.default_rng(1)
    xs = rng.random((5, n)).astype(np.float32)
    ys = np.empty_like(xs)
    check(lib.knnx_spmv_host_batch(op.h, 5, C.c_void_p(xs.ctypes.data), C.c_void_p(ys.ctypes.data)))
    for s in range(5):
        want = oracle.spmv(rp, cols, vals.astype(np.float64), xs[s].astype(np.float64))
        assert scale_rel(ys[s], want) <= 1e-5
        assert np.array_equal(ys[s], op.spmv_host(xs[s]))
    xd = torch.from_numpy(xs).cuda()
    yd = torch.empty_like(xd)
    check(lib.knnx_spmv_batch_dev(op.h, 5, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr())))
    ctx.sync()
    assert np.array_equal(yd.cpu().numpy(), ys)


@pytest.mark.parametrize("pinned", [True, False])
def test_host_entry_points_pinned_buffers(ctx, small, pinned):
    """Pinned (mapped) caller buffers take the zero-copy path -- the multiply
    stores y straight into host memory while x comes in by the copy engine;
    pageable buffers use both copy engines.  Results equal the device path bit
    for bit, with ragged sizes (n not a multiple of 4)."""
    import torch

    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import check, lib
    for n_rows in (small.cfg.n, small.cfg.n - 3):
        csr = small.csr_c.row_block(0, n_rows)
        rp, cols, vals = csr.export()
        n = small.cfg.n
        op = api.Operator.from_csr(ctx, n_rows, n, rp, cols, vals, api.CLUSTER)
        rng = np.random.default_rng(2)
        steps = 19
        xs = torch.from_numpy(rng.random((steps, n)).astype(np.float32))
        ys = torch.full((steps, n_rows), -1.0)
        if pinned:
            xs, ys = xs.pin_memory(), ys.pin_memory()
        check(lib.knnx_spmv_host_batch(op.h, steps, C.c_void_p(xs.data_ptr()),
                                       C.c_void_p(ys.data_ptr())))
        y1 = torch.full((n_rows,), -1.0)
        if pinned:
            y1 = y1.pin_memory()
        for s in range(steps):
            yd = torch.empty(n_rows, device="cuda")
            op.spmv(xs[s].cuda(), yd)
            ctx.sync()
            assert torch.equal(ys[s], yd.cpu())
            check(lib.knnx_spmv_host(op.h, C.c_void_p(xs[s].data_ptr()), C.c_void_p(y1.data_ptr())))
            assert torch.equal(y1, yd.cpu())


def test_context_destroyed_before_its_operators():
    """Garbage collectors may finalise a context before its operators: the
    context stays alive until its last operator is destroyed."""
    import gc

    from paper_1709_03671_b200 import api
    c = api.Context(0)
    op = api.Operator.from_csr(c, 2, 2, np.array([0, 1, 2]), np.array([1, 0]),
                               np.array([2.0, 3.0], np.float32), api.CLUSTER)
    c.close()
    assert np.array_equal(op.spmv_host(np.array([1.0, 10.0], np.float32)), [20.0, 3.0])
    op.close()
    # a cycle holding both, collected in arbitrary order
    c2 = api.Context(0)
    op2 = api.Operator.from_csr(c2, 1, 1, np.array([0, 1]), np.array([0]), None, api.CLUSTER)
    cyc = {"c": c2, "op": op2}
    cyc["self"] = cyc
    del c2, op2, cyc
    gc.collect()


def test_copy_async(ctx):
    import torch

    from paper_1709_03671_b200._lib import KnnxError, check, lib
    h = torch.arange(4096, dtype=torch.float32).pin_memory()
    d = torch.empty(4096, device="cuda")
    check(lib.knnx_copy_async(ctx.h, C.c_void_p(d.data_ptr()), C.c_void_p(h.data_ptr()), 4096 * 4))
    back = torch.zeros(4096).pin_memory()
    check(lib.knnx_copy_async(ctx.h, C.c_void_p(back.data_ptr()), C.c_void_p(d.data_ptr()), 4096 * 4))
    ctx.sync()
    assert torch.equal(back, h)
    with pytest.raises(KnnxError):
        check(lib.knnx_copy_async(ctx.h, C.c_void_p(d.data_ptr()), C.c_void_p(h.data_ptr()), 6))


def test_validation_errors(ctx):
    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import KnnxError
    rp = np.array([0, 2, 3], np.int64)
    with pytest.raises(KnnxError) as e:  # columns must be strictly ascending
        api.Operator.from_csr(ctx, 2, 2, rp, np.array([1, 0, 1], np.int32), None)
    assert e.value.name == "DuplicateEntry"
    with pytest.raises(KnnxError) as e:
        api.Operator.from_csr(ctx, 2, 2, rp, np.array([0, 5, 1], np.int32), None)
    assert e.value.name == "OutOfBounds"
    with pytest.raises(KnnxError) as e:
        api.Operator.from_csr(ctx, 2, 2, rp, np.array([0, 1, 1], np.int32),
                              np.array([1.0, np.inf, 2.0], np.float32))
    assert e.value.name == "NonFiniteValue"
    op = api.Operator.from_csr(ctx, 2, 3, rp, np.array([0, 1, 1], np.int32),
                               np.array([1.0, 2.0, 3.0], np.float32))
    with pytest.raises(KnnxError) as e:  # t-SNE needs a square operator
        op.tsne_host(np.zeros((2, 2), np.float32))
    assert e.value.name == "NotSquare"
    sq = api.Operator.from_csr(ctx, 2, 2, rp, np.array([0, 1, 1], np.int32), None)
    with pytest.raises(KnnxError) as e:  # stationary multiply without values
        sq.spmv_host(np.ones(2, np.float32))
    assert e.value.name == "InvalidArgument"
    with pytest.raises(KnnxError) as e:
        sq.meanshift_host(np.zeros((2, 1), np.float32), np.zeros((2, 1), np.float32), -1.0)
    assert e.value.name == "NonPositiveBandwidth"


def test_empty_and_tiny_operators(ctx, oracle):
    """Edge cases the reference tests: empty rows, a single entry, one row."""
    from paper_1709_03671_b200 import api
    rp = np.array([0, 0, 1, 1], np.int64)  # rows 0 and 2 empty
    for order in (api.ORIGINAL, api.CLUSTER):
        op = api.Operator.from_csr(ctx, 3, 3, rp, np.array([2], np.int32),
                                   np.array([2.5], np.float32), order)
        assert np.array_equal(op.spmv_host(np.array([1.0, 2.0, 4.0], np.float32)), [0.0, 10.0, 0.0])
    op = api.Operator.from_csr(ctx, 0, 0, np.array([0], np.int64), np.array([], np.int32),
                               np.array([], np.float32), api.CLUSTER)
    assert op.spmv_host(np.array([], np.float32)).size == 0
