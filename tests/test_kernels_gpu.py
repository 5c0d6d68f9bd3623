"""Raw C-ABI kernel launchers (include/amsp_c.h, "kernels" section; SURVEY
§8 row b2): amsp_k_synth_grad, amsp_k_upcast_scale, amsp_k_rs_upcast_scale,
amsp_k_ag_downcast and amsp_k_adamw on device buffers, bit-exact against the
CPU oracle / an IEEE binary32 numpy restatement of the same op sequence."""
import ctypes as C

import numpy as np
import pytest

from oracle import cpu as O
from paper_2311_00257_b200 import _native as N
from paper_2311_00257_b200.engine import DEFAULT_SEED

pytestmark = pytest.mark.gpu


def _bf16_to_f32(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


def _f32_to_bf16(f):
    u = f.astype(np.float32).view(np.uint32)
    return ((u + (((u >> 16) & 1) + 0x7FFF)) >> 16).astype(np.uint16)


def _dev(arr):
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda()


def _host(t, dtype):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy().view(dtype)


def test_synth_grad_matches_oracle(cuda):
    import torch
    n, start = 100_003, 12_345
    out = torch.empty(n, dtype=torch.int16, device="cuda")
    N.check(N.lib().amsp_k_synth_grad(out.data_ptr(), start, n, DEFAULT_SEED, 3, 1, None))
    assert np.array_equal(_host(out, np.uint16), O.grads(start, n, DEFAULT_SEED, 3, 1))


# off = 0 / 8: 16-byte aligned buffers (128-bit vector path + ragged tail);
# off = 17: misaligned (element path). Both must give identical bits.
@pytest.mark.parametrize("off", [0, 8, 17])
@pytest.mark.parametrize("W", [1, 2, 3, 5, 8])
def test_upcast_and_rs_upcast_scale(cuda, off, W):
    import torch
    n = 70_001
    srcs = [O.grads(0, n + off, DEFAULT_SEED, 1, r) for r in range(W)]
    dev = [_dev(s.view(np.int16)) for s in srcs]
    scale = np.float32(1.0 / W)
    # single source
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    N.check(N.lib().amsp_k_upcast_scale(dev[0].data_ptr() + 2 * off, out.data_ptr(), n,
                                        float(scale), None))
    want1 = _bf16_to_f32(srcs[0][off:]) * scale
    assert np.array_equal(_host(out, np.float32).view(np.uint32), want1.view(np.uint32))
    # W sources, fixed rank order, then the scale
    ptrs = (C.c_void_p * W)(*[d.data_ptr() for d in dev])
    N.check(N.lib().amsp_k_rs_upcast_scale(ptrs, W, off, out.data_ptr(), n, float(scale), None))
    acc = _bf16_to_f32(srcs[0][off:])
    for r in range(1, W):
        acc = (acc + _bf16_to_f32(srcs[r][off:])).astype(np.float32)
    want = (acc * scale).astype(np.float32)
    assert np.array_equal(_host(out, np.float32).view(np.uint32), want.view(np.uint32))
    with pytest.raises(N.InvalidConfig):
        N.check(N.lib().amsp_k_rs_upcast_scale(ptrs, 9, 0, out.data_ptr(), n, 1.0, None))


@pytest.mark.parametrize("off", [0, 8, 3])
@pytest.mark.parametrize("nd", [1, 3, 8])
def test_ag_downcast_into_every_destination(cuda, off, nd):
    import torch
    n = 50_005
    rng = np.random.default_rng(7)
    src = rng.standard_normal(n).astype(np.float32)
    dsts = [torch.zeros(n + off, dtype=torch.int16, device="cuda") for _ in range(nd)]
    ptrs = (C.c_void_p * nd)(*[d.data_ptr() for d in dsts])
    N.check(N.lib().amsp_k_ag_downcast(_dev(src).data_ptr(), n, ptrs, nd, off, None))
    want = _f32_to_bf16(src)
    for d in dsts:
        got = _host(d, np.uint16)
        assert np.array_equal(got[off:], want) and not got[:off].any()


def test_raw_kernels_empty_is_noop(cuda):
    import torch
    out = torch.full((4,), 7.0, device="cuda")
    src = torch.zeros(4, dtype=torch.int16, device="cuda")
    ptrs = (C.c_void_p * 1)(src.data_ptr())
    N.check(N.lib().amsp_k_upcast_scale(src.data_ptr(), out.data_ptr(), 0, 1.0, None))
    N.check(N.lib().amsp_k_rs_upcast_scale(ptrs, 1, 0, out.data_ptr(), 0, 1.0, None))
    N.check(N.lib().amsp_k_ag_downcast(out.data_ptr(), 0, ptrs, 1, 0, None))
    torch.cuda.synchronize()
    assert out.eq(7.0).all() and not src.any()


@pytest.mark.parametrize("bf16_grad", [True, False])
@pytest.mark.parametrize("n", [33_333, 7, 4096 * 37])
def test_adamw_flat_matches_oracle_step(cuda, bf16_grad, n):
    """amsp_k_adamw over a contiguous shard == the oracle's AMSP step with one
    rank (grad scale 1), three steps (vector path + ragged tail, tail only,
    several grid strides)."""
    import torch
    h = O.hyper()
    master = np.array([O.master_init(DEFAULT_SEED, i) for i in range(n)], np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    dm, dmm, dv = _dev(master), _dev(m), _dev(v)
    dp = torch.empty(n, dtype=torch.int16, device="cuda")
    params = np.zeros(n, np.uint16)
    seg = [(0, 0, n)]
    for t in (1, 2, 3):
        g = O.grads(0, n, DEFAULT_SEED, t, 0)
        dg = _dev(g.view(np.int16)) if bf16_grad else _dev(_bf16_to_f32(g))
        N.check(N.lib().amsp_k_adamw(dg.data_ptr(), int(bf16_grad), dm.data_ptr(),
                                     dmm.data_ptr(), dv.data_ptr(), dp.data_ptr(), n, t,
                                     h.lr, h.beta1, h.beta2, h.eps, h.weight_decay, 1.0, None))
        O.step([g], seg, master, m, v, [params], O.scalars(t, 1, h))
    for got, want in ((dm, master), (dmm, m), (dv, v)):
        assert np.array_equal(_host(got, np.uint32), want.view(np.uint32))
    assert np.array_equal(_host(dp, np.uint16), params)
