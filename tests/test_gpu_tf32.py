"""The tf32 input path (north star a12: "bf16/tf32 in, fp32 accumulate").

A pose net whose spec says `input tf32` (netspec.spec(input_dtype="tf32"))
feeds conv1_1 the fp32 frames as tf32 tensor-core operands (kind::tf32,
conv_first.cu) instead of bf16: x - 0.5 and the first layer's weights are
rounded to 10 mantissa bits (cvt.rna) instead of 7. Every later layer is bf16
as before. Checked against the CPU oracle with the same tf32 rounding, per
layer at the tolerances of test_gpu_posenet.py, and against an fp64
conv1_1 on the unrounded inputs, where it must be closer than the bf16 net.
"""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

H, W, NB = 64, 96, 2


@pytest.fixture(scope="module")
def nets():
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec, synth_posenet_weights
    be = B200Backend(0)
    s32 = netspec.spec(input_dtype="tf32")
    s16 = netspec.spec()
    h32 = be.register_model(make_model("openpose", s32, b"", netspec.COCO_DIVISOR))
    h16 = be.register_model(make_model("openpose", s16, b"", netspec.COCO_DIVISOR))
    assert h32 != h16  # the spec (and so the digest) differs
    blob = synth_posenet_weights(s32)
    assert np.array_equal(blob, synth_posenet_weights(s16))  # same weights, only the input precision differs
    layers = netspec.coco_layers()
    raw = netspec.split_weights(layers, blob)
    frame = Frame(Dims(1, 3 * NB, H, W), O.batched_frame(W, H, NB, seed=7))
    yield dict(be=be, h32=h32, h16=h16, layers=layers, raw=raw, frame=frame)
    be.close()


def ulp_bf16(x):
    x = np.abs(x).astype(np.float32)
    return np.exp2(np.floor(np.log2(np.maximum(x, 1e-30))) - 7)


def test_spec_rejects_unknown_input():
    from paper_2103_04930_b200 import netspec
    with pytest.raises(ValueError):
        netspec.spec(input_dtype="fp8")


def test_tf32_takes_the_unfused_first_layer(nets):
    be, h, d = nets["be"], nets["h32"], nets["frame"].dims
    # conv12 (kinds 2/3 on layers 0/1) is bf16-only: the tf32 net runs conv_first + conv1_2
    assert be.layer_fusion(h, d, 0)[0] not in (2, 3)
    assert be.layer_fusion(nets["h16"], d, 0)[0] == 2


def test_tf32_input_as_the_layer_sees_it(nets):
    be, h, f = nets["be"], nets["h32"], nets["frame"]
    lin, _ = be.layer_io(h, f, 0)
    x = f.data.reshape(NB, 3, H, W).transpose(0, 2, 3, 1) - np.float32(0.5)
    assert lin.tobytes() == O.tf32_round(x.astype(np.float32)).tobytes()


def test_tf32_first_layers_parity(nets):
    be, h, f, layers, raw = nets["be"], nets["h32"], nets["frame"], nets["layers"], nets["raw"]
    for i in (0, 1, 2):
        lin, lout = be.layer_io(h, f, i)
        w, b, sl = raw[i]
        w = O.tf32_round(w) if i == 0 else O.bf16_round(w)
        ref = O.conv2d_nhwc(lin, w, b, relu=layers[i].act, round_bf16=True, slope=sl)
        if lout.shape[1] * 2 == lin.shape[1]:  # conv1_2 with the fused pool
            ref = O.maxpool2_nhwc(ref)
        err = np.linalg.norm(lout - ref) / np.linalg.norm(ref)
        assert err <= 1e-3, (layers[i].name, err)
        tol = ulp_bf16(ref) + 1e-4 * float(np.abs(ref).max())
        assert not (np.abs(lout - ref) > tol).any(), layers[i].name


def test_tf32_conv1_1_closer_to_fp64(nets):
    """conv1_1 against a float64 conv on the unrounded frames and weights: the
    tf32 net's error is little more than its bf16 output rounding; the bf16
    path (emulated by the oracle: its conv1_1 output only exists inside conv12)
    adds the bf16 rounding of frames and weights."""
    be, f, layers, raw = nets["be"], nets["frame"], nets["layers"], nets["raw"]
    x = (f.data.reshape(NB, 3, H, W).transpose(0, 2, 3, 1) - np.float32(0.5)).astype(np.float32)
    w, b, sl = raw[0]
    act = layers[0].act
    exact = O.conv2d_nhwc(x, w.astype(np.float32), b, relu=act, round_bf16=False, slope=sl)
    bf16_path = O.conv2d_nhwc(O.bf16_round(x), O.bf16_round(w), b, relu=act, round_bf16=True, slope=sl)
    _, tf32_out = be.layer_io(nets["h32"], f, 0)
    e32 = np.linalg.norm(tf32_out - exact) / np.linalg.norm(exact)
    e16 = np.linalg.norm(bf16_path - exact) / np.linalg.norm(exact)
    assert e32 < 0.8 * e16, (e32, e16)


def test_tf32_forward_close_to_bf16(nets):
    be, f = nets["be"], nets["frame"]
    a = be.forward(nets["h32"], f).data
    b = be.forward(nets["h16"], f).data
    assert np.isfinite(a).all()
    assert np.max(np.abs(a - b)) <= 2e-2 * np.max(np.abs(b))
