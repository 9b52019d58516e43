"""Wire-protocol behaviour of the B200 server's C++ state machine (CPU).

Runs the product server (avec::server::Server, libavec_host.so) over the
test-only CPU stub backend (tests/native/stub_server.cpp) and drives it with
(a) the UNMODIFIED reference client (oracle/_ref/ref_client, built from
/root/reference) and (b) a hand-driven raw peer, mirroring
proj/tests/test_client_server.cpp and test_cli.cpp.
"""
import json
import pathlib
import struct
import subprocess
import time

import numpy as np
import pytest

import oracle_lib as O
import wire_client as W

ROOT = pathlib.Path(__file__).resolve().parent.parent
# AVEC_STUB_BIN: another build of the stub server (e.g. the ThreadSanitizer
# one from `make tsan`)
STUB = pathlib.Path(__import__("os").environ.get("AVEC_STUB_BIN", ROOT / "build" / "avec_stub_server"))
REF_CLIENT = ROOT / "oracle" / "_ref" / "ref_client"


def _ensure_built():
    if not STUB.exists():
        subprocess.run(["make", "-C", str(ROOT), "build/avec_stub_server"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture()
def server(tmp_path):
    _ensure_built()
    log = tmp_path / "events.jsonl"
    srv = W.ServerProc([str(STUB), "--log", str(log)])
    srv.log = log
    yield srv
    srv.stop()


def events(srv):
    return [json.loads(l) for l in srv.log.read_text().splitlines() if l.strip()]


def ref_client(endpoint, *args):
    if not REF_CLIENT.exists():
        pytest.skip("reference client not built (needs /root/reference at build time)")
    r = subprocess.run([str(REF_CLIENT), "--endpoint", endpoint, *args], capture_output=True, text=True,
                       timeout=300)
    return r.returncode, json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_client_bit_identical_and_byte_account(server):
    # test_client_server.cpp:66-85 (remote == local) and :488-503 (transfer+36 per cycle)
    rc, out = ref_client(server.endpoint, "--width", "80", "--height", "48", "--frames", "6",
                         "--check-mockpose")
    assert rc == 0 and out["ok"] and out["mismatches"] == 0 and out["byte_account_bad"] == 0
    assert not out["cache_hit"]
    rc, out2 = ref_client(server.endpoint, "--width", "80", "--height", "48", "--frames", "2",
                          "--check-mockpose")
    assert rc == 0 and out2["cache_hit"]  # global model cache across sessions
    names = [e["event"] for e in events(server)]
    assert "model_stored" in names and "model_hit" in names


def test_batched_frame_folds_into_channels(server):
    rc, out = ref_client(server.endpoint, "--width", "64", "--height", "32", "--batch", "4", "--frames", "3",
                         "--check-mockpose", "--divisor", str(192.0 / 57.0))
    assert rc == 0 and out["mismatches"] == 0


def test_negotiation_byte_account(server):
    # test_client_server.cpp:87-108: cold = 37 + upload sent / 74 received; warm 37/37
    s, w, c = b"\x01\x02\x03", b"\x04" * 100, 2.0
    dg = W.model_digest(s, w, c)
    p = W.Peer(server.port)
    p.handshake()
    p.send(W.model_check(dg))
    assert p.recv_msg() == ("model_needed", dg)
    up = W.model_upload(s, w, c)
    p.send(up)
    assert p.recv_msg() == ("model_ack", dg)
    assert len(W.model_check(dg)) == 37 and len(up) == 5 + 32 + 8 + 4 + 1 + 4 + 3 + 8 + 100
    p.close()


def test_version_mismatch_acks_own_version_then_closes(server):
    p = W.Peer(server.port)
    p.send(W.hello(2))
    assert p.recv_msg() == ("hello_ack", struct.pack("<I", 1))  # server.cpp:183-195
    assert p.closed()


def test_first_message_must_be_hello(server):
    p = W.Peer(server.port)
    p.send(W.model_check(b"\x00" * 32))
    assert p.expect_error()[0] == W.WIRE_ERRORS["protocol"]
    assert p.closed()


def test_frame_before_model_is_unknown_model(server):
    p = W.Peer(server.port)
    p.handshake()
    p.send(W.frame_data(np.ones(8)))
    assert p.expect_error()[0] == W.WIRE_ERRORS["unknown_model"]
    assert p.closed()


def _ready(server, c=2.0):
    p = W.Peer(server.port)
    p.handshake()
    s, w = b"\x09\x08", b"\x07" * 16
    p.send(W.model_upload(s, w, c))
    assert p.recv_msg()[0] == "model_ack"
    return p


@pytest.mark.parametrize("bad", [
    [W.resolution(4, 2)],                                            # Resolution before FrameData
    [W.frame_data(np.ones(8)), W.frame_size(8)],                     # FrameSize before Resolution
    [W.frame_data(np.ones(8)), W.resolution(3, 1)],                  # 3 does not divide 8
    [W.frame_data(np.ones(8)), W.resolution(4, 2), W.frame_size(9)],  # FrameSize disagrees
    [W.frame_data(np.ones(8)), W.frame_data(np.ones(8))],            # FrameData repeated
    [W.frame_data(np.ones(8)), W.model_check(b"\x00" * 32)],         # ModelCheck inside a cycle
    [W.hello()],                                                     # unexpected Hello
])
def test_cycle_order_violations_are_protocol_errors(server, bad):
    # server.cpp:280-292, 325-333
    p = _ready(server)
    for b in bad:
        p.send(b)
    assert p.expect_error()[0] == W.WIRE_ERRORS["protocol"]
    assert p.closed()


def test_full_cycle_result_matches_oracle(server):
    p = _ready(server, c=2.0)
    data = np.arange(1, 33, dtype=np.float32)
    p.send(W.frame_data(data) + W.resolution(8, 4) + W.frame_size(32))
    tag, payload = p.recv_msg()
    assert tag == "forward_result"
    cs, heat = W.forward_result(payload)
    assert cs >= 0 and heat.tobytes() == O.mockpose_forward(data, 2.0).tobytes()
    # a second cycle on the same session (the cycle state resets)
    p.send(W.frame_data(data * 2) + W.resolution(8, 4) + W.frame_size(32))
    tag, payload = p.recv_msg()
    assert W.forward_result(payload)[1].tobytes() == O.mockpose_forward(data * 2, 2.0).tobytes()


def test_byte_split_and_coalesced_messages(server):
    # test_client_server.cpp:413-439: reassembly across arbitrary TCP chunking
    p = _ready(server)
    data = np.linspace(-1, 1, 48, dtype=np.float32)
    blob = W.frame_data(data) + W.resolution(6, 8) + W.frame_size(48)
    for i in range(0, len(blob), 7):
        p.send(blob[i:i + 7])
    tag, payload = p.recv_msg()
    assert W.forward_result(payload)[1].tobytes() == O.mockpose_forward(data, 2.0).tobytes()


def test_unknown_tag_poisons_and_closes(server):
    p = _ready(server)
    p.send(struct.pack("<IB", 1, 0x7f))
    assert p.expect_error()[0] == W.WIRE_ERRORS["protocol"]
    assert p.closed()


def test_malformed_payload_poisons_and_closes(server):
    p = _ready(server)
    p.send(W.frame(W.TAGS["resolution"], struct.pack("<I", 5)))  # 4 bytes, needs 8
    code, msg = p.expect_error()
    assert code == W.WIRE_ERRORS["protocol"] and "malformed" in msg
    assert p.closed()


def test_zero_length_frame_is_malformed(server):
    p = W.Peer(server.port)
    p.handshake()
    p.send(struct.pack("<I", 0))
    assert p.expect_error()[0] == W.WIRE_ERRORS["protocol"]


def test_upload_digest_mismatch(server):
    p = W.Peer(server.port)
    p.handshake()
    p.send(W.model_upload(b"\x01", b"\x02", 2.0, digest=b"\x00" * 32))
    assert p.expect_error()[0] == W.WIRE_ERRORS["protocol"]


def test_invalid_model_rejected(server):
    p = W.Peer(server.port)
    p.handshake()
    p.send(W.model_upload(b"", b"\x02", 2.0))  # empty structure (backend.cpp:72-73)
    assert p.expect_error()[0] == W.WIRE_ERRORS["invalid_model"]
    assert p.closed()


def test_peer_error_is_logged_and_closes(server):
    p = W.Peer(server.port)
    p.handshake()
    p.send(W.error_msg(7, b"client gave up"))
    assert p.closed()
    evs = events(server)
    assert any(e["event"] == "peer_error" and "internal: client gave up" in e.get("detail", "") for e in evs)


def test_too_large_upload(tmp_path):
    _ensure_built()
    srv = W.ServerProc([str(STUB), "--max-model-bytes", "64"])
    try:
        p = W.Peer(srv.port)
        p.handshake()
        p.send(W.model_upload(b"\x01" * 10, b"\x02" * 100, 2.0))
        assert p.expect_error()[0] == W.WIRE_ERRORS["too_large"]
        assert p.closed()
    finally:
        srv.stop()


def test_session_limit_busy(tmp_path):
    # test_client_server.cpp:133-154
    _ensure_built()
    log = tmp_path / "e.jsonl"
    srv = W.ServerProc([str(STUB), "--max-sessions", "1", "--log", str(log)])
    try:
        a = W.Peer(srv.port)
        a.handshake()
        b = W.Peer(srv.port)
        assert b.expect_error()[0] == W.WIRE_ERRORS["busy"]
        assert b.closed()
    finally:
        srv.stop()
    names = [json.loads(l)["event"] for l in log.read_text().splitlines()]
    assert "rejected_busy" in names and names[-1] == "server_stopped"


def test_concurrent_clients_isolation(server):
    # acceptance criterion 8: 4 clients, distinct models, every result exact
    procs = []
    for k in range(4):
        procs.append(subprocess.Popen(
            [str(REF_CLIENT), "--endpoint", server.endpoint, "--width", "64", "--height", "64",
             "--frames", "10", "--seed", str(100 + 1000 * k), "--divisor", str(1.5 + 0.5 * k),
             "--model-seed", str(7000 + k), "--weights-bytes", "32768", "--check-mockpose"],
            stdout=subprocess.PIPE, text=True))
    outs = [json.loads(p.communicate(timeout=300)[0].strip()) for p in procs]
    assert all(o["ok"] and o["mismatches"] == 0 for o in outs)
    stored = [e for e in events(server) if e["event"] == "model_stored"]
    assert len(stored) == 4


def test_shutdown_drains_and_logs(server):
    p = _ready(server)
    out = server.stop()
    assert "shutting down" in out
    names = [e["event"] for e in events(server)]
    assert names[-1] == "server_stopped" and "session_open" in names


def _stub(*args):
    _ensure_built()
    return W.ServerProc([str(STUB), "--print-forward-log", *args])


def _forward_log(out: str):
    line = next(l for l in out.splitlines() if l.startswith("forward_log "))
    threads = next(int(l.split()[1]) for l in out.splitlines() if l.startswith("session_threads "))
    return json.loads(line[len("forward_log "):]), threads


def test_fifo_dispatch_order_with_parallel_workers():
    """The reference's FIFO contract (harness.cpp:676-681: forward_log()[i].
    arrival_seq == i, written at server.cpp:98-101) on the multi-worker
    server: 6 concurrent reference clients, a backend with 3 parallel workers
    whose forwards take a jittered 0-8 ms so completions interleave. The log is
    written at dequeue under the queue lock, so it still reads 0, 1, 2, ..."""
    srv = _stub("--concurrency", "3", "--jitter-ms", "8")
    try:
        procs = [subprocess.Popen([str(REF_CLIENT), "--endpoint", srv.endpoint, "--width", "64", "--height", "32",
                                   "--frames", "15", "--seed", str(100 + k), "--check-mockpose"],
                                  stdout=subprocess.PIPE, text=True) for k in range(6)]
        outs = [json.loads(p.communicate(timeout=300)[0].strip().splitlines()[-1]) for p in procs]
        assert all(o["ok"] and o["mismatches"] == 0 for o in outs)
    finally:
        out = srv.stop()
    log, _ = _forward_log(out)
    assert len(log) == 6 * 15
    assert [e[0] for e in log] == list(range(len(log)))
    assert len({e[1] for e in log}) == 6  # all six sessions dispatched


def test_forward_log_bounded_and_sessions_reaped():
    """A long-lived server keeps at most forward_log_cap log entries (the
    newest, still consecutive) and joins the threads of ended sessions when
    new ones arrive instead of holding one per session ever opened."""
    srv = _stub("--forward-log-cap", "5")
    try:
        for k in range(10):
            rc, o = ref_client(srv.endpoint, "--width", "16", "--height", "8", "--frames", "2", "--seed", str(k),
                               "--check-mockpose")
            assert rc == 0 and o["mismatches"] == 0
    finally:
        out = srv.stop()
    log, threads = _forward_log(out)
    assert [e[0] for e in log] == list(range(15, 20))
    assert threads <= 2, threads


def test_pipelined_cycle_speculation():
    """Receive/compute overlap (north star subsystem 2) on the server side: a
    FrameData of the previous cycle's size starts the cycle on the backend
    pipeline with the previous model and dims, before Resolution (which the
    wire sends AFTER the frame, server.cpp:272-292) can confirm them. A
    Resolution with other dims, or a new model, must drop the guess; every
    reply must equal the reference's segment means for the cycle's own model.
    The stub pipeline computes with the GUESSED model, so a guess the server
    failed to drop would show up as a wrong result."""
    _ensure_built()
    srv = W.ServerProc([str(STUB), "--print-forward-log", "--pipeline"])
    try:
        p = _ready(srv, c=2.0)
        rng = np.random.default_rng(5)

        def cycle(w, h, c):
            data = rng.random(w * h * 3, dtype=np.float32)
            p.send(W.frame_data(data) + W.resolution(w, h) + W.frame_size(data.size))
            tag, payload = p.recv_msg()
            assert tag == "forward_result", tag
            got = W.forward_result(payload)[1]
            assert got.tobytes() == O.mockpose_forward(data, c).tobytes(), (w, h, c)
            time.sleep(0.05)  # the helper thread prepares the next cycle's pipeline

        for _ in range(3):
            cycle(64, 32, 2.0)      # cycles 2, 3 speculate and finish on the pipeline
        cycle(32, 64, 2.0)          # same size, other dims: speculated, then dropped
        cycle(32, 64, 2.0)          # speculates with the new dims
        s2, w2 = b"\x05\x06", b"\x01" * 8
        p.send(W.model_upload(s2, w2, 4.0))
        assert p.recv_msg()[0] == "model_ack"
        cycle(32, 64, 4.0)          # new model: no speculation
        cycle(32, 64, 4.0)          # speculates with the new model
        p.close()
    finally:
        out = srv.stop()
    line = next(l for l in out.splitlines() if l.startswith("pipeline "))
    counts = dict(zip(line.split()[1::2], map(int, line.split()[2::2])))
    # speculation starts once the helper thread has prepared the pipeline for
    # the session's last cycle; normally cycles 2, 3, 4 (dropped), 5 and 7
    # speculate. A loaded host can make the helper miss a cycle, so the counts
    # are bounds; a guess that is neither dropped nor finished never passes,
    # and a guess that was not dropped shows up as a wrong result above
    assert counts["begins"] == counts["finishes"] + counts["aborts"], counts
    assert counts["aborts"] <= 1 and 2 <= counts["finishes"] <= 4, counts
    assert counts["feeds"] >= counts["begins"]


def test_pipelined_session_disconnect_mid_frame():
    """A session whose speculative cycle is streaming when the client vanishes
    (half a FrameData sent, then close) must not take the server down or leak
    into the next session; the next session's cycles stay exact."""
    _ensure_built()
    srv = W.ServerProc([str(STUB), "--print-forward-log", "--pipeline"])
    try:
        p = _ready(srv, c=2.0)
        data = np.random.default_rng(1).random(64 * 32 * 3, dtype=np.float32)
        p.send(W.frame_data(data) + W.resolution(64, 32) + W.frame_size(data.size))
        assert p.recv_msg()[0] == "forward_result"
        import time
        time.sleep(0.2)  # the helper thread prepares the pipeline
        frame = W.frame_data(data)
        p.send(frame[: len(frame) // 2])  # speculation starts, then the peer goes away
        time.sleep(0.1)
        p.close()
        q = _ready(srv, c=2.0)
        for k in range(3):
            d = np.random.default_rng(10 + k).random(64 * 32 * 3, dtype=np.float32)
            q.send(W.frame_data(d) + W.resolution(64, 32) + W.frame_size(d.size))
            tag, payload = q.recv_msg()
            assert tag == "forward_result"
            assert W.forward_result(payload)[1].tobytes() == O.mockpose_forward(d, 2.0).tobytes()
        q.close()
        assert srv.p.poll() is None
    finally:
        out = srv.stop()
    line = next(l for l in out.splitlines() if l.startswith("pipeline "))
    counts = dict(zip(line.split()[1::2], map(int, line.split()[2::2])))
    assert counts["begins"] >= 2  # the abandoned speculation and the second session's
