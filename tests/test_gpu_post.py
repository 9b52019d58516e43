"""Upsample / NMS kernels against the oracle on their own inputs (bit-exact),
across the code paths launch_upsample and launch_nms pick: x8 interior +
border kernels, the general power-of-two kernel (x16), the generic kernel
(x2, x3), and NMS on widths that are / are not multiples of four."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def be():
    from paper_2103_04930_b200 import B200Backend
    b = B200Backend(0)
    yield b
    b.close()


@pytest.mark.parametrize("scale,h,w", [(8, 5, 7), (8, 46, 82), (16, 6, 9), (2, 9, 14), (3, 4, 8)])
def test_upsample_bitexact(be, scale, h, w):
    import torch
    rng = np.random.default_rng(scale * 100 + w)
    planes = 3
    x = rng.standard_normal((planes, h, w)).astype(np.float32)
    d_in = torch.from_numpy(x).cuda()
    d_out = torch.empty((planes, h * scale, w * scale), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    be.upsample_device(d_in.data_ptr(), planes, h, w, scale, d_out.data_ptr())
    got = d_out.cpu().numpy()
    for p in range(planes):
        assert got[p].tobytes() == O.upsample_plane(x[p], scale).tobytes(), p


@pytest.mark.parametrize("h,w", [(37, 64), (20, 50), (64, 1312)])
def test_nms_bitexact(be, h, w):
    import torch
    rng = np.random.default_rng(h * w)
    planes = 4
    # blocky field with plateaus (ties must not count as peaks) and spikes
    x = np.round(rng.random((planes, h, w)) * 8).astype(np.float32) / 8
    thr, maxp = 0.3, 512
    d_x = torch.from_numpy(x).cuda()
    d_cnt = torch.zeros(planes, dtype=torch.int32, device="cuda")
    d_pk = torch.zeros((planes, maxp, 5), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    be.nms_device(d_x.data_ptr(), planes, h, w, thr, maxp, d_cnt.data_ptr(), d_pk.data_ptr())
    cnt, pk = d_cnt.cpu().numpy(), d_pk.cpu().numpy()
    for p in range(planes):
        xy, ref, sc = O.nms_plane(x[p], thr, maxp)
        n = len(sc)
        assert cnt[p] == n and n > 0
        assert np.array_equal(pk[p, :n, 0:2].astype(np.int32), xy)
        assert pk[p, :n, 2:4].tobytes() == ref.tobytes() and pk[p, :n, 4].tobytes() == sc.tobytes()


@pytest.mark.parametrize("planes,h,w", [(3, 5, 7), (144, 46, 82), (2, 92, 164), (2, 1, 3), (2, 3, 256), (2, 4, 257)])
def test_upsample_nms_fused_bitexact(be, planes, h, w):
    """avec_upsample_nms_device = avec_upsample_device then avec_nms_device,
    bit for bit, and against the oracle: the fused kernel (w <= 256) and the
    two-launch fallback (w = 257). Fields with plateaus after the upsample
    (ties), corner spikes (the row-end groups), and +inf / NaN source pixels."""
    import torch
    rng = np.random.default_rng(planes * 1000 + h * w)
    x = (np.round(rng.random((planes, h, w)) * 6) / 6).astype(np.float32)
    x[0, 0, 0] = 5.0  # spike at the corner (row-end group 0)
    x[-1, h - 1, w - 1] = 7.0  # and at the far corner (group w - 1)
    if planes > 3:  # fused vs split only: NaN payloads differ between the GPU and x86 oracle
        x[1, h // 2, w // 2] = np.inf
        x[2, h // 2, 1] = np.nan
    thr, maxp = 0.35, 96
    d_x = torch.from_numpy(x).cuda()
    up_a = torch.full((planes, 8 * h, 8 * w), 3.0, dtype=torch.float32, device="cuda")
    up_b = torch.empty_like(up_a)
    ca = torch.zeros(planes, dtype=torch.int32, device="cuda")
    cb = torch.zeros_like(ca)
    pa = torch.zeros((planes, maxp, 5), dtype=torch.float32, device="cuda")
    pb = torch.zeros_like(pa)
    torch.cuda.synchronize()
    be.upsample_nms_device(d_x.data_ptr(), planes, h, w, 8, thr, maxp, up_a.data_ptr(), ca.data_ptr(), pa.data_ptr())
    be.upsample_device(d_x.data_ptr(), planes, h, w, 8, up_b.data_ptr())
    be.nms_device(up_b.data_ptr(), planes, 8 * h, 8 * w, thr, maxp, cb.data_ptr(), pb.data_ptr())
    ua, ub = up_a.cpu().numpy(), up_b.cpu().numpy()
    assert ua.tobytes() == ub.tobytes()
    assert np.array_equal(ca.cpu().numpy(), cb.cpu().numpy())
    assert pa.cpu().numpy().tobytes() == pb.cpu().numpy().tobytes()
    cnt, pk = ca.cpu().numpy(), pa.cpu().numpy()
    for p in sorted({0, planes - 1}):
        ref_up = O.upsample_plane(x[p], 8)
        assert ua[p].tobytes() == ref_up.tobytes(), p
        xy, ref, sc = O.nms_plane(ref_up, thr, maxp)
        n = len(sc)
        assert cnt[p] == n, p
        assert np.array_equal(pk[p, :n, 0:2].astype(np.int32), xy)
        assert pk[p, :n, 2:4].tobytes() == ref.tobytes() and pk[p, :n, 4].tobytes() == sc.tobytes()
    if h >= 5:  # (tiny planes are all plateaus after the upsample)
        assert cnt.sum() > 0


def test_upsample_nms_rejects_other_scales(be):
    import torch
    from paper_2103_04930_b200 import AvecError
    d = torch.zeros((1, 4, 4), dtype=torch.float32, device="cuda")
    o = torch.zeros((1, 16, 16), dtype=torch.float32, device="cuda")
    c = torch.zeros(1, dtype=torch.int32, device="cuda")
    pk = torch.zeros((1, 4, 5), dtype=torch.float32, device="cuda")
    with pytest.raises(AvecError):
        be.upsample_nms_device(d.data_ptr(), 1, 4, 4, 4, 0.1, 4, o.data_ptr(), c.data_ptr(), pk.data_ptr())
