"""The real B200 server (bin/avec-server) driven by the UNMODIFIED reference
client — the drop-in claim (SURVEY.md §4 implication: acceptance 2/8,
test_cli.cpp:301-317 digest equality) — plus pose-net cycles over the wire.
"""
import hashlib
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


@pytest.fixture(scope="module")
def server(tmp_path_factory):
    log = tmp_path_factory.mktemp("srv") / "events.jsonl"
    srv = W.ServerProc([str(SERVER), "--log", str(log)])
    srv.log = log
    yield srv
    out = srv.stop()
    assert "shutting down" in out


def ref_client(endpoint, *args):
    r = subprocess.run([str(REF_CLIENT), "--endpoint", endpoint, *args], capture_output=True, text=True,
                       timeout=600)
    return r.returncode, json.loads(r.stdout.strip().splitlines()[-1])


def test_banner(server):
    assert server.banner.startswith("listening on 127.0.0.1:") and "(backend b200" in server.banner


def test_reference_client_mockpose_bit_identical(server):
    # every cycle memcmp'd against the reference's own mockpose_forward
    rc, out = ref_client(server.endpoint, "--width", "656", "--height", "368", "--frames", "5",
                         "--check-mockpose")
    assert rc == 0 and out["mismatches"] == 0 and out["byte_account_bad"] == 0


def test_reference_client_golden_digest(server, golden):
    # 368x368 frame 0 seed 7 c=3.368421 -> SURVEY.md §8(c) digest, through the wire
    rc, out = ref_client(server.endpoint, "--width", "368", "--height", "368", "--frames", "1",
                         "--check-mockpose", "--dump", "/tmp/avec_dump_368.bin")
    assert rc == 0
    heat = np.fromfile("/tmp/avec_dump_368.bin", dtype=np.float32)
    assert hashlib.sha256(heat.tobytes()).hexdigest() == \
        "46372e4b33930c40ffd16e0ee001b51d329737dc2ed5a93cef35e7ec4d49de23"


def test_reference_client_batched_c2(server, golden):
    rc, out = ref_client(server.endpoint, "--width", "656", "--height", "368", "--batch", "8", "--frames", "2",
                         "--check-mockpose", "--divisor", repr(192.0 / 57.0))
    assert rc == 0 and out["mismatches"] == 0 and out["expect_cycle_bytes"] == 30055308 + 36


def test_posenet_over_the_wire_equals_c_abi(server, tmp_path):
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
    spec = tmp_path / "spec.txt"
    spec.write_bytes(netspec.spec())
    h, w, b = 64, 96, 2
    rc, out = ref_client(server.endpoint, "--structure", str(spec), "--divisor", repr(netspec.COCO_DIVISOR),
                         "--width", str(w), "--height", str(h), "--batch", str(b), "--frames", "2",
                         "--dump", str(tmp_path / "heat.bin"), "--name", "openpose_coco")
    assert rc == 0 and out["ok"] and out["byte_account_bad"] == 0
    wire_out = np.fromfile(tmp_path / "heat.bin", dtype=np.float32).reshape(2, -1)
    be = B200Backend(0)
    hd = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    for cyc in range(2):
        frame = O.batched_frame(w, h, b, seed=7, first=cyc * b)
        local = be.forward(hd, Frame(Dims(1, 3 * b, h, w), frame)).data
        assert local.size == b * 57 * (h // 8) * (w // 8)
        assert wire_out[cyc].tobytes() == local.tobytes()
    be.close()


def test_tf32_posenet_over_the_wire_equals_c_abi(server, tmp_path):
    """An `input tf32` net uploaded by the unmodified reference client (the
    spec rides in the model structure) replies what the C-ABI computes."""
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
    s32 = netspec.spec(input_dtype="tf32")
    spec = tmp_path / "spec32.txt"
    spec.write_bytes(s32)
    h, w, b = 64, 96, 2
    rc, out = ref_client(server.endpoint, "--structure", str(spec), "--divisor", repr(netspec.COCO_DIVISOR),
                         "--width", str(w), "--height", str(h), "--batch", str(b), "--frames", "1",
                         "--dump", str(tmp_path / "heat32.bin"), "--name", "openpose_coco_tf32")
    assert rc == 0 and out["ok"] and out["byte_account_bad"] == 0
    wire_out = np.fromfile(tmp_path / "heat32.bin", dtype=np.float32)
    be = B200Backend(0)
    hd = be.register_model(make_model("openpose_coco_tf32", s32, b"", netspec.COCO_DIVISOR))
    local = be.forward(hd, Frame(Dims(1, 3 * b, h, w), O.batched_frame(w, h, b, seed=7))).data
    assert wire_out.tobytes() == local.tobytes()
    be.close()


def test_c1_reference_client_posenet_368(server, tmp_path):
    """BASELINE configs[0] (C1): the unmodified reference client drives the COCO
    pose net through our server, one 368x368 frame, batch 1. The wire reply is
    the C-ABI result bit for bit and matches the CPU oracle chain within 2e-2
    (bf16 rounding flips propagate through 92 layers); the NMS peaks of its
    upsampled heatmaps are bit-exact against the oracle NMS."""
    import torch
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec, synth_posenet_weights
    spec = tmp_path / "spec.txt"
    spec.write_bytes(netspec.spec())
    h = w = 368
    rc, out = ref_client(server.endpoint, "--structure", str(spec), "--divisor", repr(netspec.COCO_DIVISOR),
                         "--width", str(w), "--height", str(h), "--batch", "1", "--frames", "1",
                         "--dump", str(tmp_path / "heat.bin"), "--name", "openpose_coco")
    assert rc == 0 and out["ok"] and out["byte_account_bad"] == 0
    wire_out = np.fromfile(tmp_path / "heat.bin", dtype=np.float32)
    assert wire_out.size == 57 * 46 * 46 == 120612  # K at C1
    frame = O.batched_frame(w, h, 1, seed=7)
    be = B200Backend(0)
    hd = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    local = be.forward(hd, Frame(Dims(1, 3, h, w), frame)).data
    assert wire_out.tobytes() == local.tobytes()
    layers = netspec.coco_layers()
    wb = [(O.bf16_round(wt), b, sl) for wt, b, sl in netspec.split_weights(layers, synth_posenet_weights(netspec.spec()))]
    want = O.coco_chain(frame.reshape(1, 3, h, w), layers, wb)
    err = np.linalg.norm(local - want) / np.linalg.norm(want)
    assert err < 2e-2, err
    # keypoint candidates: x8 upsample + 3x3 NMS on the 18 part heatmaps
    planes = np.ascontiguousarray(local.reshape(57, 46, 46)[:18])
    d_in = torch.from_numpy(planes).cuda()
    d_up = torch.empty((18, h, w), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    be.upsample_device(d_in.data_ptr(), 18, 46, 46, 8, d_up.data_ptr())
    up = d_up.cpu().numpy()
    thr = float(np.quantile(up, 0.5))
    maxp = 96
    d_cnt = torch.zeros(18, dtype=torch.int32, device="cuda")
    d_pk = torch.zeros((18, maxp, 5), dtype=torch.float32, device="cuda")
    be.nms_device(d_up.data_ptr(), 18, h, w, thr, maxp, d_cnt.data_ptr(), d_pk.data_ptr())
    cnt, pk = d_cnt.cpu().numpy(), d_pk.cpu().numpy()
    for p in range(18):
        assert up[p].tobytes() == O.upsample_plane(planes[p], 8).tobytes(), p
        xy, ref, sc = O.nms_plane(up[p], thr, maxp)
        n = len(sc)
        assert cnt[p] == n
        assert np.array_equal(pk[p, :n, 0:2].astype(np.int32), xy)
        assert pk[p, :n, 2:4].tobytes() == ref.tobytes() and pk[p, :n, 4].tobytes() == sc.tobytes()
    be.close()


def test_posenet_bad_resolution_is_internal_error(server, tmp_path):
    from paper_2103_04930_b200 import netspec
    s = netspec.spec()
    p = W.Peer(server.port)
    p.handshake()
    p.send(W.model_upload(s, b"", netspec.COCO_DIVISOR, name=b"openpose"))
    assert p.recv_msg()[0] == "model_ack"
    data = np.zeros(3 * 30 * 20, np.float32)  # 30 x 20: not divisible by 8
    p.send(W.frame_data(data) + W.resolution(30, 20) + W.frame_size(data.size))
    assert p.expect_error()[0] == W.WIRE_ERRORS["internal"]


def test_concurrent_reference_clients_fifo_and_isolation(server):
    procs = []
    for k in range(4):
        procs.append(subprocess.Popen(
            [str(REF_CLIENT), "--endpoint", server.endpoint, "--width", "128", "--height", "96",
             "--frames", "12", "--seed", str(100 + 1000 * k), "--divisor", str(1.5 + 0.5 * k),
             "--model-seed", str(7000 + k), "--weights-bytes", "32768", "--check-mockpose"],
            stdout=subprocess.PIPE, text=True))
    outs = [json.loads(p.communicate(timeout=300)[0].strip()) for p in procs]
    assert all(o["ok"] and o["mismatches"] == 0 for o in outs)


def test_loadgen_posenet_throughput(server):
    r = subprocess.run([str(LOADGEN), "--endpoint", server.endpoint, "--clients", "2", "--steps", "6",
                        "--warmup", "2", "--batch", "8"], capture_output=True, text=True, timeout=600)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["ok"] and out["fps"] > 50


def test_reference_server_with_b200_plugin():
    """Plugin-level drop-in: the reference's OWN Server (built from its sources)
    with the B200 engine behind accelfwd::backend::Backend via the C-ABI shim
    (oracle/ref_drivers/b200_shim.hpp = INTEGRATION.md), driven by the
    reference client: results bit-identical to its local MockPose."""
    exe = ROOT / "oracle" / "_ref" / "ref_b200_server"
    srv = W.ServerProc([str(exe)])
    try:
        assert "(backend b200:0)" in srv.banner
        rc, out = ref_client(srv.endpoint, "--width", "656", "--height", "368", "--batch", "2",
                             "--frames", "3", "--check-mockpose")
        assert rc == 0 and out["mismatches"] == 0 and out["byte_account_bad"] == 0
    finally:
        srv.stop()


def test_reference_server_b200_plugin_survives_bad_shape():
    """A pose-net frame the engine rejects (367 rows: not divisible by 8) comes
    from the client; through the shim it must surface as accelfwd::Error ->
    ErrorMsg internal (server.cpp:313-318), not as an exception that escapes
    the reference's session thread and terminates the server. A second
    session afterwards still gets served."""
    from paper_2103_04930_b200 import netspec
    exe = ROOT / "oracle" / "_ref" / "ref_b200_server"
    srv = W.ServerProc([str(exe)])
    try:
        s = netspec.spec()
        for hgt, ok in ((367, False), (368, True)):
            p = W.Peer(srv.port, timeout=120)
            p.handshake()
            p.send(W.model_upload(s, b"", netspec.COCO_DIVISOR, name=b"openpose"))
            assert p.recv_msg()[0] == "model_ack"
            data = np.zeros(3 * hgt * 64, np.float32)
            p.send(W.frame_data(data) + W.resolution(64, hgt) + W.frame_size(data.size))
            if ok:
                tag, payload = p.recv_msg()
                assert tag == "forward_result"
                assert W.forward_result(payload)[1].size == 57 * (hgt // 8) * 8
            else:
                assert p.expect_error()[0] == W.WIRE_ERRORS["internal"]
            p.close()
        assert srv.p.poll() is None
    finally:
        srv.stop()


def test_split_policy_server(tmp_path):
    srv = W.ServerProc([str(SERVER), "--policy", "split", "--slots", "1"])
    try:
        r = subprocess.run([str(LOADGEN), "--endpoint", srv.endpoint, "--clients", "1", "--steps", "3",
                            "--warmup", "1", "--batch", "4", "--width", "128", "--height", "96"],
                           capture_output=True, text=True, timeout=600)
        assert json.loads(r.stdout.strip().splitlines()[-1])["ok"]
    finally:
        srv.stop()
