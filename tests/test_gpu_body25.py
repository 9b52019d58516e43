"""GPU parity of the BODY_25 family (PReLU, dense blocks, 4 PAF + 2 heatmap
stages) against the CPU oracle — same tolerances as tests/test_gpu_posenet.py:
per layer ||gpu-oracle||/||oracle|| <= 1e-3 and every element within one bf16
ulp + 1e-4*max|oracle| (intermediate layers); fp32 outputs to 1e-3 relative."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

H, W, NB = 64, 96, 2


@pytest.fixture(scope="module")
def b25():
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec, synth_posenet_weights
    be = B200Backend(0)
    s = netspec.spec("openpose_body25")
    h = be.register_model(make_model("body25", s, b"", netspec.BODY25_DIVISOR))
    layers = netspec.body25_layers()
    wb = [(O.bf16_round(w), b, sl) for w, b, sl in netspec.split_weights(layers, synth_posenet_weights(s))]
    frame = Frame(Dims(1, 3 * NB, H, W), O.batched_frame(W, H, NB, seed=3))
    yield dict(be=be, h=h, layers=layers, wb=wb, frame=frame)
    be.close()


def ulp_bf16(x):
    x = np.abs(x).astype(np.float32)
    return np.exp2(np.floor(np.log2(np.maximum(x, 1e-30))) - 7)


def test_layer_table(b25):
    from paper_2103_04930_b200 import netspec
    assert b25["be"].num_layers(b25["h"]) == 114
    assert netspec.macs_per_pixel(b25["layers"]) == 594970


def test_output_size_and_law(b25):
    be, h = b25["be"], b25["h"]
    out = be.forward(h, b25["frame"]).data
    assert out.size == NB * 78 * (H // 8) * (W // 8)
    assert np.isfinite(out).all()


def test_all_layers_parity(b25):
    be, h, layers = b25["be"], b25["h"], b25["layers"]
    finals = {i for i, L in enumerate(layers) if L.name in ("Mconv7_stage3_L2", "Mconv7_stage1_L1")}
    for i, L in enumerate(layers):
        kind, src = be.layer_fusion(h, b25["frame"].dims, i)
        if kind == 2:  # Mconv6 of a fused head: checked through its Mconv7
            continue
        lin, lout = be.layer_io(h, b25["frame"], i)
        w, b, sl = b25["wb"][i]
        final = i in finals
        x = lin
        if kind == 3:  # fused head: chain Mconv6 (bf16 intermediate) from the head input
            w6, b6, s6 = b25["wb"][src]
            x = O.conv2d_nhwc(lin, w6, b6, relu=layers[src].act, round_bf16=True, slope=s6)
        ref = O.conv2d_nhwc(x, w, b, relu=L.act, round_bf16=not final, slope=sl)
        if lout.shape[1] * 2 == lin.shape[1]:  # the plan fuses this layer's 2x2 max-pool
            ref = O.maxpool2_nhwc(ref)
        err = np.linalg.norm(lout - ref) / max(np.linalg.norm(ref), 1e-30)
        assert err <= 1e-3, (L.name, err)
        if not final and kind != 3:
            tol = ulp_bf16(ref) + 1e-4 * float(np.abs(ref).max())
            assert not (np.abs(lout - ref) > tol).any(), L.name


def test_wire_layout_heat_then_paf(b25):
    be, h = b25["be"], b25["h"]
    out = be.forward(h, b25["frame"]).data.reshape(NB, 78, H // 8, W // 8)
    names = [L.name for L in b25["layers"]]
    _, heat = be.layer_io(h, b25["frame"], names.index("Mconv7_stage1_L1"))
    _, paf = be.layer_io(h, b25["frame"], names.index("Mconv7_stage3_L2"))
    assert np.array_equal(out[:, :26], heat.transpose(0, 3, 1, 2))
    assert np.array_equal(out[:, 26:], paf.transpose(0, 3, 1, 2))


def test_split_batch_equals_whole(b25):
    """Frame groups (the multi-GPU split) give the same bits as one batch."""
    from paper_2103_04930_b200 import Dims, Frame
    be, h = b25["be"], b25["h"]
    whole = be.forward(h, b25["frame"]).data.reshape(NB, -1)
    per = b25["frame"].data.reshape(NB, -1)
    for i in range(NB):
        one = be.forward(h, Frame(Dims(1, 3, H, W), per[i])).data
        assert one.tobytes() == whole[i].tobytes()


_SINGLE_CTA_HEADS = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
import oracle_lib as O
from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
be = B200Backend(0, slots=1)
h = be.register_model(make_model("body25", netspec.spec("openpose_body25"), b"", netspec.BODY25_DIVISOR))
w, hgt, nb = int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
f = Frame(Dims(1, 3 * nb, hgt, w), O.batched_frame(w, hgt, nb, seed=9))
np.save(sys.argv[2], be.forward(h, f).data)
be.close()
"""


def test_pair_heads_bit_identical_to_single_cta(b25, tmp_path):
    """BODY_25's stage heads run on CTA pairs (conv_head2: M = 256 MMAs, the
    input tile resident across the c6 blocks). Each output element sees the
    same bf16 operands in the same K order as the single-CTA kernel, so the
    whole forward is bit-identical to AVEC_HEAD2=0 (run in a subprocess). A
    200x80 frame gives an odd number (3) of 128-pixel tiles per image at the head
    level, so the pair's second CTA also runs a tile wholly past the image."""
    import os
    import pathlib
    import subprocess
    import sys
    from paper_2103_04930_b200 import Dims, Frame
    be, h = b25["be"], b25["h"]
    w, hgt, nb = 200, 80, 3
    frame = Frame(Dims(1, 3 * nb, hgt, w), O.batched_frame(w, hgt, nb, seed=9))
    out = be.forward(h, frame).data
    root = str(pathlib.Path(__file__).resolve().parent.parent)
    dst = tmp_path / "single.npy"
    subprocess.run([sys.executable, "-c", _SINGLE_CTA_HEADS, root, str(dst), str(w), str(hgt), str(nb)],
                   env=dict(os.environ, AVEC_HEAD2="0"), check=True, timeout=600)
    assert out.tobytes() == np.load(dst).tobytes()


def test_k16_tail_skip_bit_identical(b25, tmp_path):
    """The pixel-major kernel skips the zero-weight K16 steps of a layer's last
    64-channel chunk (96-channel dense-block inputs, 288-channel block concats,
    the mapped stage input). Those steps only add exact zeros, so the forward
    is bit-identical to issuing them (AVEC_K16TAIL=0, in a subprocess)."""
    import os
    import pathlib
    import subprocess
    import sys
    from paper_2103_04930_b200 import Dims, Frame
    be, h = b25["be"], b25["h"]
    w, hgt, nb = 200, 80, 3
    frame = Frame(Dims(1, 3 * nb, hgt, w), O.batched_frame(w, hgt, nb, seed=9))
    out = be.forward(h, frame).data
    root = str(pathlib.Path(__file__).resolve().parent.parent)
    dst = tmp_path / "full_k.npy"
    subprocess.run([sys.executable, "-c", _SINGLE_CTA_HEADS, root, str(dst), str(w), str(hgt), str(nb)],
                   env=dict(os.environ, AVEC_K16TAIL="0"), check=True, timeout=600)
    assert out.tobytes() == np.load(dst).tobytes()
