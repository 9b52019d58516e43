"""Multi-GPU product path; needs a box with >= 2 GPUs
(`gpurun --gpus 2`), skipped otherwise.

avec-server --policy split cuts every batched cycle into contiguous frame
groups (avec_frame_groups, the partition tests/test_sharding.py checks on a
gloo world), runs them on the GPUs concurrently and writes each group's slice
of the batch-major reply. Frames are independent (batch folded into channels,
/root/reference/proj/src/server.cpp:297-301), so:
  * C5 (BODY_25, 32 x 1312x736 over 2 GPUs): the reply driven by the
    unmodified reference client equals the 1-GPU forward of the whole batch
    bit for bit (the 16-frame plans pick the same kernels as the 32-frame one);
  * C2 (COCO, 8 x 656x368): each GPU's 4-frame group equals that group run on
    one GPU bit for bit; the 4-frame plan runs its 7x7 convs split-K (64 tiles
    for 148 SMs), so against the 8-frame plan it agrees to the end-to-end
    tolerance, not bitwise.
"""
import json
import pathlib
import subprocess

import numpy as np
import pytest

import oracle_lib as O
import wire_client as W

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parent.parent
SERVER = ROOT / "paper_2103_04930_b200" / "bin" / "avec-server"
LOADGEN = ROOT / "paper_2103_04930_b200" / "bin" / "avec-loadgen"
REF_CLIENT = ROOT / "oracle" / "_ref" / "ref_client"


def _gpus():
    try:
        from paper_2103_04930_b200.backend import device_count
        return device_count()
    except Exception:  # no GPU / no driver (CPU collection)
        return 0


needs2 = pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")


def _wire_forward(endpoint, spec_path, divisor, w, h, batch, dump, name):
    r = subprocess.run([str(REF_CLIENT), "--endpoint", endpoint, "--structure", str(spec_path), "--divisor",
                        repr(divisor), "--width", str(w), "--height", str(h), "--batch", str(batch), "--frames", "1",
                        "--dump", str(dump), "--name", name, "--cycle-timeout", "600"],
                       capture_output=True, text=True, timeout=900)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and out["ok"] and out["byte_account_bad"] == 0, out
    return np.fromfile(dump, dtype=np.float32)


@needs2
def test_split_policy_c5_bit_identical_to_one_gpu(tmp_path):
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
    fam, w, h, nb = "openpose_body25", 1312, 736, 32
    spec = tmp_path / "b25.spec"
    spec.write_bytes(netspec.spec(fam))
    srv = W.ServerProc([str(SERVER), "--policy", "split", "--devices", "0,1", "--slots", "1"])
    try:
        assert "split" in srv.banner
        got = _wire_forward(srv.endpoint, spec, netspec.BODY25_DIVISOR, w, h, nb, tmp_path / "o.bin", fam)
    finally:
        srv.stop()
    be = B200Backend(0, slots=1)
    hd = be.register_model(make_model(fam, netspec.spec(fam), b"", netspec.BODY25_DIVISOR))
    want = be.forward(hd, Frame(Dims(1, 3 * nb, h, w), O.batched_frame(w, h, nb, seed=7))).data
    be.close()
    assert got.size == nb * 78 * (h // 8) * (w // 8)
    assert got.tobytes() == want.tobytes()


@needs2
def test_split_policy_c2_groups_bit_identical(tmp_path):
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
    from paper_2103_04930_b200.sharding import frame_groups
    fam, w, h, nb = "openpose_coco", 656, 368, 8
    spec = tmp_path / "coco.spec"
    spec.write_bytes(netspec.spec(fam))
    srv = W.ServerProc([str(SERVER), "--policy", "split", "--devices", "0,1", "--slots", "1"])
    try:
        got = _wire_forward(srv.endpoint, spec, netspec.COCO_DIVISOR, w, h, nb, tmp_path / "o.bin", fam)
    finally:
        srv.stop()
    frames = O.batched_frame(w, h, nb, seed=7).reshape(nb, -1)
    per = 57 * (h // 8) * (w // 8)
    be = B200Backend(1, slots=1)  # the second GPU recomputing every group: devices agree bit for bit
    hd = be.register_model(make_model(fam, netspec.spec(fam), b"", netspec.COCO_DIVISOR))
    for first, n in frame_groups(nb, 2):
        sub = be.forward(hd, Frame(Dims(1, 3 * n, h, w), frames[first:first + n].ravel())).data
        assert got[first * per:(first + n) * per].tobytes() == sub.tobytes(), first
    whole = be.forward(hd, Frame(Dims(1, 3 * nb, h, w), frames.ravel())).data
    be.close()
    assert np.linalg.norm(got - whole) / np.linalg.norm(whole) < 1e-2


@needs2
def test_session_policy_pins_and_serves(tmp_path):
    """C4's placement: session k on GPU (k-1) mod 2. Four concurrent
    reference clients, every MockPose result bit-exact against the reference's
    own local computation, then a posenet load through loadgen."""
    srv = W.ServerProc([str(SERVER), "--policy", "session", "--devices", "0,1", "--slots", "1"])
    try:
        assert "session" in srv.banner
        procs = [subprocess.Popen([str(REF_CLIENT), "--endpoint", srv.endpoint, "--width", "656", "--height", "368",
                                   "--batch", "2", "--frames", "6", "--seed", str(100 + k), "--check-mockpose"],
                                  stdout=subprocess.PIPE, text=True) for k in range(4)]
        outs = [json.loads(p.communicate(timeout=300)[0].strip().splitlines()[-1]) for p in procs]
        assert all(o["ok"] and o["mismatches"] == 0 for o in outs)
        r = subprocess.run([str(LOADGEN), "--endpoint", srv.endpoint, "--clients", "4", "--steps", "6",
                            "--warmup", "2", "--batch", "8"], capture_output=True, text=True, timeout=600)
        assert json.loads(r.stdout.strip().splitlines()[-1])["ok"]
    finally:
        srv.stop()


@needs2
def test_pipelined_sessions_on_two_gpus(tmp_path):
    """Two concurrent reference clients on a 2-GPU server (session policy:
    one session per GPU, so each GPU's pool pipelines its session's repeat
    cycles): every reply equals the 1-GPU whole-batch forward bit for bit
    (the C2 4-frame groups keep the 8-frame plan's kernels and K order)."""
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
    spec = tmp_path / "coco.spec"
    spec.write_bytes(netspec.spec())
    w, h, nb, cycles = 656, 368, 8, 4
    log = tmp_path / "events.jsonl"
    srv = W.ServerProc([str(SERVER), "--policy", "session", "--devices", "0,1", "--slots", "1", "--log", str(log)])
    try:
        procs = [subprocess.Popen([str(REF_CLIENT), "--endpoint", srv.endpoint, "--structure", str(spec), "--divisor",
                                   repr(netspec.COCO_DIVISOR), "--width", str(w), "--height", str(h), "--batch",
                                   str(nb), "--frames", str(cycles), "--seed", str(7 + k), "--dump",
                                   str(tmp_path / f"o{k}.bin"), "--name", "openpose_coco"],
                                  stdout=subprocess.PIPE, text=True) for k in range(2)]
        outs = [json.loads(p.communicate(timeout=600)[0].strip().splitlines()[-1]) for p in procs]
        assert all(o["ok"] and o["byte_account_bad"] == 0 for o in outs)
    finally:
        srv.stop()
    be = B200Backend(0, slots=1)
    hd = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    for k in range(2):
        got = np.fromfile(tmp_path / f"o{k}.bin", dtype=np.float32).reshape(cycles, -1)
        for c in range(cycles):
            frames = O.batched_frame(w, h, nb, seed=7 + k, first=c * nb)
            want = be.forward(hd, Frame(Dims(1, 3 * nb, h, w), frames)).data
            assert got[c].tobytes() == want.tobytes(), (k, c)
    be.close()
    events = [json.loads(l)["event"] for l in log.read_text().splitlines() if l.strip()]
    assert events.count("cycle_pipelined") >= 2
