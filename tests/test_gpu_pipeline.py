"""Pipelined cycles (avec_stream_*; north star subsystem 2): frames land in a
pinned buffer front to back while H2D, group compute and D2H proceed on side
streams. Results must equal the non-pipelined forward of the same frame
groups bit for bit (frames are independent, batch folded into channels,
/root/reference/proj/src/server.cpp:297-301), and the segment-mean model must
stay bit-exact against the CPU oracle (its boundaries are global, so it
computes once the frame is complete)."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def _land(stream, total, steps):
    """Report `total` bytes landing in `steps` uneven increments."""
    edges = sorted({int(total * (k / steps) ** 1.5) for k in range(1, steps)} | {total})
    for e in edges:
        stream.feed(e)


@pytest.fixture(scope="module")
def be():
    from paper_2103_04930_b200 import B200Backend
    b = B200Backend(0, slots=1)
    yield b
    b.close()


def test_pipelined_c2_equals_groups(be):
    from paper_2103_04930_b200 import Dims, Frame, PinnedBuffer, PipelineStream, make_model, netspec
    w, h, nb = 656, 368, 8
    hd = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    dims = Dims(1, 3 * nb, h, w)
    frames = O.batched_frame(w, h, nb, seed=7)
    K = be.output_elems(hd, dims)
    pin_in, pin_out = PinnedBuffer(frames.size), PinnedBuffer(K)
    pin_in.array[:] = frames
    st = PipelineStream(be)
    for steps in (1, 7, 40):
        pin_out.array[:] = np.nan
        st.begin(hd, dims, pin_in.ptr, pin_out.ptr, K)
        _land(st, frames.nbytes, steps)
        secs = st.finish()
        assert secs > 0
        got = pin_out.array.copy()
        per_frame = K // nb
        for f0, n in ((0, 4), (4, 4)):  # the stream's two frame groups
            sub = frames.reshape(nb, -1)[f0:f0 + n].ravel()
            want = be.forward(hd, Frame(Dims(1, 3 * n, h, w), sub)).data
            assert got[f0 * per_frame:(f0 + n) * per_frame].tobytes() == want.tobytes(), (steps, f0)
    whole = be.forward(hd, Frame(dims, frames)).data
    assert np.linalg.norm(got - whole) / np.linalg.norm(whole) < 1e-2
    st.close()


def test_pipelined_body25_odd_batch(be):
    """5 frames: groups of 3 and 2 (two plan sizes), BODY_25."""
    from paper_2103_04930_b200 import Dims, Frame, PinnedBuffer, PipelineStream, make_model, netspec
    w, h, nb = 128, 96, 5
    hd = be.register_model(make_model("b25", netspec.spec("openpose_body25"), b"", netspec.BODY25_DIVISOR))
    dims = Dims(1, 3 * nb, h, w)
    frames = O.batched_frame(w, h, nb, seed=3)
    K = be.output_elems(hd, dims)
    pin_in, pin_out = PinnedBuffer(frames.size), PinnedBuffer(K)
    pin_in.array[:] = frames
    st = PipelineStream(be)
    st.begin(hd, dims, pin_in.ptr, pin_out.ptr, K)
    _land(st, frames.nbytes, 9)
    st.finish()
    per = K // nb
    for f0, n in ((0, 3), (3, 2)):
        want = be.forward(hd, Frame(Dims(1, 3 * n, h, w), frames.reshape(nb, -1)[f0:f0 + n].ravel())).data
        assert pin_out.array[f0 * per:(f0 + n) * per].tobytes() == want.tobytes(), f0
    st.close()


def test_pipelined_mockpose_bit_exact_and_abort(be):
    from paper_2103_04930_b200 import Dims, PinnedBuffer, PipelineStream, make_model
    hd = be.register_model(make_model("pose-est", bytes(range(16)), b"\x01", 3.368421))
    dims = Dims(1, 24, 368, 656)
    frames = O.batched_frame(656, 368, 8, seed=7)
    K = be.output_elems(hd, dims)
    pin_in, pin_out = PinnedBuffer(frames.size), PinnedBuffer(K)
    pin_in.array[:] = frames
    st = PipelineStream(be)
    st.begin(hd, dims, pin_in.ptr, pin_out.ptr, K)
    st.feed(frames.nbytes // 3)
    st.abort()  # speculation dropped mid-frame: the next cycle starts clean
    st.begin(hd, dims, pin_in.ptr, pin_out.ptr, K)
    _land(st, frames.nbytes, 5)
    st.finish()
    assert pin_out.array.tobytes() == O.mockpose_forward(frames, 3.368421).tobytes()
    st.close()


def test_server_pipelines_repeat_cycles(tmp_path):
    """Through avec-server with the unmodified reference client: the first C2
    cycle of a session runs whole (8-frame plan); later cycles of the same
    size are pipelined while their frames arrive, as two 4-frame groups (the
    server logs `cycle_pipelined`). Each reply equals the C-ABI forward of
    those frame groups bit for bit, and here also the whole-batch forward:
    the 4-frame plan keeps every conv on the same kernels and K order, so
    every cycle is checked against both whatever path it took."""
    import pathlib
    import subprocess
    import json
    import wire_client as W
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
    root = pathlib.Path(__file__).resolve().parent.parent
    spec = tmp_path / "coco.spec"
    spec.write_bytes(netspec.spec())
    w, h, nb, cycles = 656, 368, 8, 4
    log = tmp_path / "events.jsonl"
    srv = W.ServerProc([str(root / "paper_2103_04930_b200" / "bin" / "avec-server"), "--slots", "1", "--devices", "0",
                        "--log", str(log)])
    try:
        r = subprocess.run([str(root / "oracle" / "_ref" / "ref_client"), "--endpoint", srv.endpoint, "--structure",
                            str(spec), "--divisor", repr(netspec.COCO_DIVISOR), "--width", str(w), "--height", str(h),
                            "--batch", str(nb), "--frames", str(cycles), "--dump", str(tmp_path / "o.bin"),
                            "--name", "openpose_coco"], capture_output=True, text=True, timeout=600)
        out = json.loads(r.stdout.strip().splitlines()[-1])
        assert r.returncode == 0 and out["ok"] and out["byte_account_bad"] == 0
    finally:
        srv.stop()
    got = np.fromfile(tmp_path / "o.bin", dtype=np.float32).reshape(cycles, -1)
    be = B200Backend(0, slots=1)
    hd = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    per = got.shape[1] // nb
    for c in range(cycles):
        frames = O.batched_frame(w, h, nb, seed=7, first=c * nb).reshape(nb, -1)
        whole = be.forward(hd, Frame(Dims(1, 3 * nb, h, w), frames.ravel())).data
        assert got[c].tobytes() == whole.tobytes(), c
        for f0 in (0, 4):
            grp = be.forward(hd, Frame(Dims(1, 12, h, w), frames[f0:f0 + 4].ravel())).data
            assert got[c, f0 * per:(f0 + 4) * per].tobytes() == grp.tobytes(), (c, f0)
    be.close()
    # speculation starts once a helper thread has prepared the pipeline after
    # the first cycle, so the second cycle (on a loaded box, the third) may
    # still run whole; the first never pipelines
    events = [json.loads(l)["event"] for l in log.read_text().splitlines() if l.strip()]
    assert 1 <= events.count("cycle_pipelined") <= cycles - 1


@pytest.mark.parametrize("nb", [8, 7])
def test_forward_pinned_is_two_frame_groups(be, nb):
    """avec_forward between pinned host buffers runs a multi-frame pose-net
    cycle as two frame groups whose copies overlap the other group's compute
    (engine.cu pipelined_posenet, cycles of >= 64 MB of frames): its output
    is the two groups' forwards, bit for bit (8 frames: 4 + 4; 7 frames:
    4 + 3, two plan sizes)."""
    from paper_2103_04930_b200 import Dims, Frame, PinnedBuffer, make_model, netspec
    w, h = 1312, 736  # 8 frames: 92.7 MB
    hd = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    dims = Dims(1, 3 * nb, h, w)
    frames = O.batched_frame(w, h, nb, seed=11)
    K = be.output_elems(hd, dims)
    pin_in, pin_out = PinnedBuffer(frames.size), PinnedBuffer(K)
    pin_in.array[:] = frames
    for _ in range(2):  # the second cycle reuses the slot's staging and group plans
        pin_out.array[:] = np.nan
        be.forward(hd, Frame(dims, pin_in.array), out=pin_out.array)
        got = pin_out.array.copy()
        per_frame = K // nb
        g0 = (nb + 1) // 2
        for f0, n in ((0, g0), (g0, nb - g0)):
            sub = frames.reshape(nb, -1)[f0:f0 + n].ravel()
            want = be.forward(hd, Frame(Dims(1, 3 * n, h, w), sub)).data
            assert got[f0 * per_frame:(f0 + n) * per_frame].tobytes() == want.tobytes(), f0
    pin_in.free()
    pin_out.free()
