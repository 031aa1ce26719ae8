"""tcgen05 / TMEM Gram kernel (knnx_gram_tf32_dev): C = A B^T with the
operands read as TF32 and fp32 accumulation in tensor memory.  With inputs
already representable in TF32 every product is exact in fp32, so the result
must match a float64 GEMM to fp32 accumulation rounding; ragged tile edges
(m, n not multiples of 128 / 256) included."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tf32(a):
    b = np.ascontiguousarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32)


@pytest.mark.parametrize("m,n,k", [(128, 256, 32), (300, 520, 960), (1, 7, 64), (513, 1025, 128)])
def test_gram_tf32_exact_inputs(ctx, m, n, k):
    import torch

    from paper_1709_03671_b200._lib import check, lib
    rng = np.random.default_rng(m + n + k)
    a = _tf32(rng.standard_normal((m, k)))
    b = _tf32(rng.standard_normal((n, k)))
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    cd = torch.full((m, n), np.nan, device="cuda")
    check(lib.knnx_gram_tf32_dev(ctx.h, C.c_void_p(ad.data_ptr()), m, C.c_void_p(bd.data_ptr()), n,
                                 k, k, C.c_void_p(cd.data_ptr()), n))
    ctx.sync()
    got = cd.cpu().numpy()
    want = a.astype(np.float64) @ b.astype(np.float64).T
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64).T
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - want) / scale) < 1e-6


def test_gram_tf32_fp32_inputs(ctx):
    """Full fp32 inputs: TF32 truncation of the operands, ~1e-3 relative."""
    import torch

    from paper_1709_03671_b200._lib import check, lib
    rng = np.random.default_rng(3)
    m, n, k = 256, 512, 960
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    cd = torch.empty((m, n), device="cuda")
    check(lib.knnx_gram_tf32_dev(ctx.h, C.c_void_p(ad.data_ptr()), m, C.c_void_p(bd.data_ptr()), n,
                                 k, k, C.c_void_p(cd.data_ptr()), n))
    ctx.sync()
    want = a.astype(np.float64) @ b.astype(np.float64).T
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64).T
    assert np.max(np.abs(cd.cpu().numpy() - want) / scale) < 2e-3
