"""CPU checks of the row-sampled parity machinery (no GPU).

* oracle_conv2d_rows equals the matching rows of oracle_conv2d_nhwc bit for
  bit (same arithmetic), for 1x1/3x3/7x7, ReLU/PReLU/none, rows at the image
  border (zero windows) included;
* tests/fullsize.check_layer_rows, driven by a stand-in backend that serves
  rows of oracle-computed tensors, accepts a correct layer (plain, pooled, a
  chained conv1_1+conv1_2+pool pair, a chained 1x1 head) and rejects a layer
  with one corrupted element in a sampled row.
"""
import dataclasses

import numpy as np
import pytest

import fullsize as F
import oracle_lib as O


def _rand(rng, shape, scale=1.0):
    return O.bf16_round((rng.standard_normal(shape) * scale).astype(np.float32))


@pytest.mark.parametrize("k,act", [(1, 0), (3, 1), (3, 2), (7, 1)])
def test_conv2d_rows_matches_full_tensor(k, act):
    rng = np.random.default_rng(k * 10 + act)
    n, h, w, cin, cout = 2, 9, 13, 5, 6
    x = _rand(rng, (n, h, w, cin))
    wt = _rand(rng, (cout, cin, k, k), 0.2)
    b = rng.standard_normal(cout).astype(np.float32)
    sl = rng.random(cout).astype(np.float32) * 0.3
    full = O.conv2d_nhwc(x, wt, b, relu=act, round_bf16=True, slope=sl)
    p = k // 2
    sel = [(0, 0), (0, h - 1), (1, 4), (1, 0), (0, 2)]
    zero = np.zeros((w, cin), np.float32)
    win = np.stack([np.stack([x[bi, y + d] if 0 <= y + d < h else zero for d in range(-p, p + 1)])
                    for bi, y in sel])
    rows = O.conv2d_rows(win, wt, b, relu=act, round_bf16=True, slope=sl)
    for r, (bi, y) in enumerate(sel):
        assert rows[r].tobytes() == full[bi, y].tobytes()


@dataclasses.dataclass(frozen=True)
class L:
    name: str
    cin: int
    cout: int
    k: int
    act: int
    level: int


class _FakeBackend:
    """Serves layer_rows from whole tensors computed by the oracle, the way
    the engine's plan executes the tiny net below (fusion kinds as the engine
    reports them)."""

    def __init__(self, layers, wb, frames, corrupt=None):
        self.layers, self.wb = layers, wb
        self.corrupt = corrupt
        x = O.bf16_round(frames.transpose(0, 2, 3, 1) - 0.5)
        self.t = {}
        a = O.conv2d_nhwc(x, *wb[0][:2], relu=1, round_bf16=True)
        b = O.maxpool2_nhwc(O.conv2d_nhwc(a, *wb[1][:2], relu=1, round_bf16=True))
        c = O.conv2d_nhwc(b, *wb[2][:2], relu=1, round_bf16=True)
        d = O.maxpool2_nhwc(O.conv2d_nhwc(c, *wb[3][:2], relu=1, round_bf16=True))
        e = O.conv2d_nhwc(d, *wb[4][:2], relu=1, round_bf16=True)
        f = O.conv2d_nhwc(e, *wb[5][:2], relu=0, round_bf16=False)
        # layer -> (input tensor as the plan shows it, output tensor)
        self.io = {1: (x, b), 2: (b, c), 3: (c, d), 5: (d, f)}
        self.fusion = {0: (2, 0), 1: (3, 0), 2: (0, 2), 3: (1, 3), 4: (2, 4), 5: (3, 4)}

    def layer_fusion(self, h, dims, i):
        return self.fusion[i]

    def layer_out_level(self, h, dims, i):
        return {1: 1, 2: 1, 3: 2, 5: 2}[i]

    def layer_rows(self, h, frame, i, in_sel, out_sel):
        tin, tout = self.io[i]
        zero = np.zeros(tin.shape[2:], np.float32)
        lin = np.stack([tin[b, y] if 0 <= y < tin.shape[1] else zero for b, y in in_sel])
        lout = np.stack([tout[b, y] for b, y in out_sel]).copy()
        if self.corrupt == i:
            lout[-1, 1, 0] += 0.5
        return lin, lout


def _tiny():
    layers = [L("conv1_1", 3, 8, 3, 1, 0), L("conv1_2", 8, 8, 3, 1, 0), L("conv2_1", 8, 16, 3, 1, 1),
              L("conv2_2", 16, 16, 3, 1, 1), L("Mconv6", 16, 32, 1, 1, 2), L("Mconv7", 32, 5, 1, 0, 2)]
    rng = np.random.default_rng(1)
    wb = [(_rand(rng, (l.cout, l.cin, l.k, l.k), 0.3), rng.standard_normal(l.cout).astype(np.float32) * 0.1, None)
          for l in layers]
    frames = rng.random((2, 3, 16, 24)).astype(np.float32)

    class Dims:
        batch, channels, height, width = 1, 6, 16, 24

    class Frame:
        dims = Dims()
    return layers, wb, frames, Frame()


def test_check_layer_rows_accepts_correct_layers():
    layers, wb, frames, frame = _tiny()
    be = _FakeBackend(layers, wb, frames)
    assert F.check_layer_rows(be, None, frame, layers, wb, 0, final=False) is None
    for i in (1, 2, 3):
        err, mx, n = F.check_layer_rows(be, None, frame, layers, wb, i, final=False)
        assert err == 0.0 and mx == 0.0 and n > 0, i
    err, mx, n = F.check_layer_rows(be, None, frame, layers, wb, 5, final=True)
    assert err == 0.0


@pytest.mark.parametrize("i", [2, 3])
def test_check_layer_rows_rejects_corruption(i):
    layers, wb, frames, frame = _tiny()
    be = _FakeBackend(layers, wb, frames, corrupt=i)
    with pytest.raises(AssertionError):
        F.check_layer_rows(be, None, frame, layers, wb, i, final=False)
