"""Pin the CPU oracle to the reference's own outputs (tests/golden/reference_golden.json).

Each check mirrors a reference test: test_wire.cpp:137-149 (sizing law),
test_backend.cpp:48-120 (segment means), acceptance.cpp:386-421 (brute-force
instances), plus SURVEY.md §8(c)'s frame/heatmap digests.
"""
import hashlib
import struct

import numpy as np
import pytest

import oracle_lib as O


def _d(bits_hex: str) -> float:
    return struct.unpack("<d", bytes.fromhex(bits_hex)[::-1])[0]


def test_output_elems_fixed_points(golden):
    # test_wire.cpp:137-143
    assert O.output_elems(5, 2.0) == 3
    assert O.output_elems(3, 2.0) == 2
    assert O.output_elems(10, 3.0) == 3
    assert O.output_elems(1, 3.0) == 0
    assert O.output_elems(724224, 3.368421) == 215004
    for e, cbits, k in golden["output_elems"]:
        assert O.output_elems(e, _d(cbits)) == k


def test_transfer_size_fixed_points(golden):
    # test_wire.cpp:145-149
    assert O.transfer_size(1, 3, 368, 656, 3.368421) == 3756924
    assert O.transfer_size(1, 1, 1, 1, 1.0) == 20
    assert O.transfer_size(1, 3, 100, 100, 3.368421) == 155636
    for n, c, h, w, cbits, ts in golden["transfer_size"]:
        assert O.transfer_size(n, c, h, w, _d(cbits)) == ts


def test_gen_frame_small_bitexact(golden):
    g = golden["gen_frame_small"]
    f = O.gen_frame(g["seed"], g["index"], g["w"], g["h"])
    assert f.view(np.uint32).tolist() == g["bits"]


@pytest.mark.parametrize("i", range(7))
def test_gen_frame_and_mockpose_digests(golden, i):
    g = golden["gen_frame"][i]
    f = O.gen_frame(g["seed"], g["index"], g["w"], g["h"])
    assert hashlib.sha256(f.tobytes()).hexdigest() == g["frame_sha256"]
    heat = O.mockpose_forward(f, _d(g["divisor_bits"]))
    assert heat.size == g["k"]
    assert heat[:3].view(np.uint32).tolist() == g["heat_first"]
    assert hashlib.sha256(heat.tobytes()).hexdigest() == g["heat_sha256"]


def test_survey_digests_match(golden):
    # SURVEY.md §8(c) goldens captured from the reference
    want = {(368, 368): "46372e4b33930c40ffd16e0ee001b51d329737dc2ed5a93cef35e7ec4d49de23",
            (656, 368): "68a691f92b8b59aa4a80ef0e5c115cbe2a438177091c7c34b8b17c207aed4196",
            (1312, 736): "d5e7864b36c7d14da69bab68d1fe1ed1bcc81cf8a98c53e4a809a05ee5458971"}
    for (w, h), dig in want.items():
        f = O.gen_frame(7, 0, w, h)
        heat = O.mockpose_forward(f, 3.368421)
        assert hashlib.sha256(heat.tobytes()).hexdigest() == dig


def test_batched_c2_digest(golden):
    g = golden["batched_c2"]
    f = O.batched_frame(g["w"], g["h"], g["batch"], g["seed"])
    assert hashlib.sha256(f.tobytes()).hexdigest() == g["frame_sha256"]
    heat = O.mockpose_forward(f, 192.0 / 57.0)
    assert heat.size == g["k"] == 1720032
    assert hashlib.sha256(heat.tobytes()).hexdigest() == g["heat_sha256"]


def test_segment_means_fixed_points():
    # test_backend.cpp:48-63
    m = O.segment_means(np.arange(1, 9, dtype=np.float32), 2.0)
    assert m.tolist() == [1.5, 3.5, 5.5, 7.5]
    m = O.segment_means(np.arange(1, 11, dtype=np.float32), 3.0)
    assert m.tolist() == [2.0, 5.0, 8.5]


def test_segment_means_brute_force_instances(golden):
    # acceptance.cpp:386-421 recipe, values produced by the reference itself
    for inst in golden["segment_means"]:
        data = np.array(inst["data"], np.uint32).view(np.float32)
        got = O.segment_means(data, _d(inst["divisor_bits"]))
        want = [_d(b) for b in inst["means"]]
        assert got.tolist() == want


def test_constant_invariance():
    # test_backend.cpp:97-102
    data = np.full(731, 0.5, np.float32)
    for c in (1.0, 2.0, 3.368421, 7.3):
        assert np.all(O.segment_means(data, c) == 0.5)


def test_degenerate_rejections(golden):
    # test_backend.cpp:104-120
    with pytest.raises(O.OracleError, match="degenerate_output"):
        O.segment_means(np.array([1.0], np.float32), 3.0)
    with pytest.raises(O.OracleError, match="degenerate_output"):
        O.segment_means(np.array([1, 2, 3, 4], np.float32), 0.3)
    with pytest.raises(O.OracleError, match="empty"):
        O.segment_means(np.array([], np.float32), 1.0)
    assert [d["error"] for d in golden["degenerate"]] == ["degenerate_output"] * 2


def test_synth_model_blobs(golden):
    # harness.cpp:355-370 and the model digest law wire.cpp:70-79
    for g in golden["synth_model"]:
        s, w = O.synth_blobs(g["seed"], g["structure_bytes"], g["weights_bytes"])
        assert hashlib.sha256(s).hexdigest() == g["structure_sha256"]
        assert hashlib.sha256(w).hexdigest() == g["weights_sha256"]
        c = struct.pack("<d", _d(g["divisor_bits"]))
        assert hashlib.sha256(s + w + c).hexdigest() == g["digest"]


def test_bf16_round_matches_c():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(1000).astype(np.float32) * 10
    x[:4] = [0.0, -0.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8]  # ties to even both ways
    v = O.bf16_round(x)
    for a, b in zip(x[:200], v[:200]):
        assert O.lib().oracle_bf16_round(float(a)) == b
    assert v[2] == 1.0 and v[3] == 1.0 + 2 ** -6


def test_conv_oracle_against_numpy():
    rng = np.random.default_rng(1)
    x = O.bf16_round(rng.standard_normal((2, 6, 5, 7)).astype(np.float32))
    w = rng.standard_normal((4, 7, 3, 3)).astype(np.float32)
    b = rng.standard_normal(4).astype(np.float32)
    got = O.conv2d_nhwc(x, w, b, relu=False, round_bf16=False)
    xp = np.pad(x.astype(np.float64), ((0, 0), (1, 1), (1, 1), (0, 0)))
    want = np.zeros((2, 6, 5, 4))
    for r in range(3):
        for s in range(3):
            want += np.einsum("nhwc,oc->nhwo", xp[:, r:r + 6, s:s + 5, :], w[:, :, r, s].astype(np.float64))
    want += b
    np.testing.assert_allclose(got, want.astype(np.float32), rtol=1e-6, atol=1e-6)


def test_upsample_and_nms_oracle_semantics():
    x = np.zeros((4, 5), np.float32)
    x[1, 2] = 1.0
    x[3, 4] = 0.5
    up = O.upsample_plane(x, 8)
    assert up.shape == (32, 40)
    # half-pixel centres: output (11.5 -> 12) rows around source row 1 peak
    assert up.max() == 1.0 or up.max() < 1.0 + 1e-6
    xy, ref, sc = O.nms_plane(x, 0.05, 10)
    assert xy.tolist() == [[2, 1], [4, 3]]
    assert sc.tolist() == [1.0, 0.5]
    assert ref.tolist() == [[2.0, 1.0], [4.0, 3.0]]
