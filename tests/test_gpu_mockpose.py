"""GPU parity of the reference's own model (segment means) through the C-ABI.

Bar: bit-exact. Every result is compared byte-for-byte with the CPU oracle and,
where the reference produced one, with its golden digest
(tests/golden/reference_golden.json). Mirrors proj/tests/test_backend.cpp and
acceptance.cpp criterion 9.
"""
import hashlib
import struct

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def _d(bits_hex: str) -> float:
    return struct.unpack("<d", bytes.fromhex(bits_hex)[::-1])[0]


@pytest.fixture(scope="module")
def be():
    from paper_2103_04930_b200 import B200Backend
    b = B200Backend(0)
    yield b
    b.close()


def model(divisor, tag=0):
    from paper_2103_04930_b200 import make_model
    return make_model("m", bytes([tag, 1, 2]), bytes([3, 4]), divisor)


def fwd(be, data, divisor, tag=0, dims=None):
    from paper_2103_04930_b200 import Dims, Frame
    h = be.register_model(model(divisor, tag))
    data = np.ascontiguousarray(data, np.float32)
    dims = dims or Dims(1, 1, 1, data.size)
    return be.forward(h, Frame(dims, data)).data


def test_label_and_handles(be):
    # test_backend.cpp:130-138 — idempotent per digest, ids start at 1
    assert be.label() == "b200:0"
    a = be.register_model(model(2.0, 1))
    b = be.register_model(model(2.0, 1))
    c = be.register_model(model(2.0, 2))
    assert a == b and a.id != c.id
    assert min(a.id, c.id) >= 1


def test_ids_start_at_one():
    from paper_2103_04930_b200 import B200Backend
    b = B200Backend(0, slots=1)
    assert b.register_model(model(3.0, 9)).id == 1
    b.close()


def test_rejects_bad_models_and_unknown_handles(be):
    from paper_2103_04930_b200 import AvecError, Dims, Frame, ModelDescriptor, ModelHandle, model_digest
    bad = ModelDescriptor("m", b"\x01", b"", -1.0, model_digest(b"\x01", b"", -1.0))
    with pytest.raises(AvecError) as e:
        be.register_model(bad)
    assert e.value.name == "invalid_model"
    empty = ModelDescriptor("m", b"", b"\x01", 2.0, model_digest(b"", b"\x01", 2.0))
    with pytest.raises(AvecError) as e:
        be.register_model(empty)
    assert e.value.name == "invalid_model"
    with pytest.raises(AvecError) as e:
        be.forward(ModelHandle(987654), Frame(Dims(1, 1, 1, 4), np.ones(4, np.float32)))
    assert e.value.name == "unknown_model"
    h = be.register_model(model(2.0, 3))
    with pytest.raises(ValueError):
        be.forward(h, Frame(Dims(1, 1, 2, 4), np.ones(4, np.float32)))


def test_degenerate_output(be):
    from paper_2103_04930_b200 import AvecError
    with pytest.raises(AvecError) as e:
        fwd(be, [1.0], 3.0)
    assert e.value.name == "degenerate_output"
    with pytest.raises(AvecError) as e:
        fwd(be, [1, 2, 3, 4], 0.3)
    assert e.value.name == "degenerate_output"


def test_fixed_points(be):
    # test_backend.cpp:48-63
    assert fwd(be, np.arange(1, 9), 2.0).tolist() == [1.5, 3.5, 5.5, 7.5]
    assert fwd(be, np.arange(1, 11), 3.0).tolist() == [2.0, 5.0, 8.5]
    for c in (1.0, 2.0, 3.368421, 7.3):  # constant invariance :97-102
        assert np.all(fwd(be, np.full(731, 0.5), c) == 0.5)


@pytest.mark.parametrize("i", range(7))
def test_reference_golden_digests(be, golden, i):
    from paper_2103_04930_b200 import Dims, Frame
    g = golden["gen_frame"][i]
    f = O.gen_frame(g["seed"], g["index"], g["w"], g["h"])
    h = be.register_model(model(_d(g["divisor_bits"]), 7))
    heat = be.forward(h, Frame(Dims(1, 3, g["h"], g["w"]), f)).data
    assert heat.size == g["k"]
    assert hashlib.sha256(heat.tobytes()).hexdigest() == g["heat_sha256"]


def test_batched_c2_golden(be, golden):
    from paper_2103_04930_b200 import Dims, Frame
    g = golden["batched_c2"]
    f = O.batched_frame(656, 368, 8)
    h = be.register_model(model(192.0 / 57.0, 8))
    heat = be.forward(h, Frame(Dims(1, 24, 368, 656), f)).data
    assert hashlib.sha256(heat.tobytes()).hexdigest() == g["heat_sha256"]


def test_brute_force_instances(be, golden):
    for inst in golden["segment_means"]:
        data = np.array(inst["data"], np.uint32).view(np.float32)
        c = _d(inst["divisor_bits"])
        want = np.array([_d(b) for b in inst["means"]]).astype(np.float32)
        assert fwd(be, data, c).tobytes() == want.tobytes()


def test_random_against_oracle(be):
    rng = np.random.default_rng(0x0BACE1E5)
    for _ in range(300):
        e = int(rng.integers(1, 20000))
        c = 1.0 if e == 1 else float(rng.uniform(1.0, min(float(e), 64.0)))
        data = rng.uniform(-8, 8, e).astype(np.float32)
        k = O.output_elems(e, c)
        if k < 1 or k > e:
            continue
        assert fwd(be, data, c).tobytes() == O.mockpose_forward(data, c).tobytes()


@pytest.mark.parametrize("c", [1.7, 2.46, 3.37, 5.5, 7.9])
def test_extreme_values(be, c):
    """Random float bit patterns over the whole exponent range, plus zeros of
    both signs, infinities and NaNs: the short-segment division (segmean.cu,
    Markstein's correction step) and its __ddiv_rn fallback for non-finite
    sums must match the reference's sum / n bit for bit (NaNs: same positions)."""
    rng = np.random.default_rng(int(c * 1000))
    bits = rng.integers(0, 2**32, 200000, dtype=np.uint64).astype(np.uint32)
    data = bits.view(np.float32).copy()
    data[~np.isfinite(data)] = 1.5
    special = rng.integers(0, data.size, 400)
    data[special[:100]] = np.inf
    data[special[100:200]] = -np.inf
    data[special[200:300]] = np.nan
    data[special[300:350]] = -0.0
    data[special[350:]] = 0.0
    got, want = fwd(be, data, c), O.mockpose_forward(data, c)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    fin = ~np.isnan(want)
    assert got[fin].tobytes() == want[fin].tobytes()


@pytest.mark.parametrize("c", [1.0, 47.5, 100.0, 1000.0, 4096.0])
def test_wide_segments(be, c):
    # widths above the shared-memory staging bound take the direct kernel
    data = np.random.default_rng(1).standard_normal(3 * 8192).astype(np.float32)
    assert fwd(be, data, c).tobytes() == O.mockpose_forward(data, c).tobytes()


def test_pinned_and_pageable_agree(be):
    from paper_2103_04930_b200 import Dims, Frame, PinnedBuffer
    f = O.batched_frame(656, 368, 2)
    h = be.register_model(model(3.368421, 11))
    d = Dims(1, 6, 368, 656)
    a = be.forward(h, Frame(d, f)).data
    pin_in = PinnedBuffer(f.size)
    pin_in.array[:] = f
    pin_out = PinnedBuffer(a.size)
    t = []
    be.forward(h, Frame(d, pin_in.array), out=pin_out.array, timing=t)
    assert pin_out.array.tobytes() == a.tobytes() == O.mockpose_forward(f, 3.368421).tobytes()
    assert t and 0 < t[0] < 5.0


def test_large_frame_c5_shape(be):
    # C5 frame size: 32 x 3 x 736 x 1312 = 92,700,672 floats (370.8 MB), c = 192/78
    from paper_2103_04930_b200 import Dims, Frame
    rng = np.random.default_rng(5)
    f = rng.random(92700672, dtype=np.float32)
    h = be.register_model(model(192.0 / 78.0, 12))
    heat = be.forward(h, Frame(Dims(1, 96, 736, 1312), f)).data
    assert heat.size == 37659648
    assert heat.tobytes() == O.mockpose_forward(f, 192.0 / 78.0).tobytes()


def test_device_resident_path(be):
    import torch
    from paper_2103_04930_b200 import Dims
    f = O.batched_frame(368, 368, 4)
    d = Dims(1, 12, 368, 368)
    h = be.register_model(model(3.368421, 13))
    k = be.output_elems(h, d)
    din = torch.from_numpy(f).cuda()
    dout = torch.empty(k, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    be.forward_device(h, d, din.data_ptr(), dout.data_ptr())
    assert dout.cpu().numpy().tobytes() == O.mockpose_forward(f, 3.368421).tobytes()


@pytest.mark.parametrize("elems,c", [(16 * 1024 * 1024 + 7, 1.0), (24_000_011, 3.368421), (5_000_000, 0.999)])
def test_overlapped_chunks_bit_exact(elems, c):
    """Pinned frames >= 16 MB take the chunked path (H2D / segment kernel /
    D2H of ~8 MB chunks cut at segment boundaries, on three streams): still
    bit-exact against the oracle, odd sizes and c < 1 (K > E rejected) included."""
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, PinnedBuffer, make_model
    be = B200Backend(0, slots=1)
    h = be.register_model(make_model("chunky", b"\x03\x04", b"", c))
    data = np.random.default_rng(elems).random(elems, dtype=np.float32)
    pin_in = PinnedBuffer(elems)
    pin_in.array[:] = data
    if c < 1.0:
        with pytest.raises(Exception):
            be.output_elems(h, Dims(1, 1, 1, elems))
        be.close()
        return
    want = O.mockpose_forward(data, c)
    pin_out = PinnedBuffer(want.size)
    be.forward(h, Frame(Dims(1, 1, 1, elems), pin_in.array), out=pin_out.array)
    assert pin_out.array.tobytes() == want.tobytes()
    be.close()
