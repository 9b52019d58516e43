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
