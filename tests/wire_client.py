"""Hand-driven AVEC protocol peer (TEST INFRASTRUCTURE).

A byte-level restatement of the reference wire format
(proj/include/accelfwd/wire.hpp:13-191, proj/src/wire.cpp) used like the
reference's RawPeer (proj/tests/test_client_server.cpp:263-302) to drive a
server through normal and malformed exchanges.
"""
from __future__ import annotations

import hashlib
import socket
import struct
import subprocess
import time

TAGS = dict(hello=1, hello_ack=2, frame_size=3, resolution=4, frame_data=5, forward_result=6,
            model_check=7, model_needed=8, model_upload=9, model_ack=10, error=11)
NAMES = {v: k for k, v in TAGS.items()}
WIRE_ERRORS = dict(protocol=1, busy=2, too_large=3, version=4, unknown_model=5, invalid_model=6, internal=7)


def frame(tag: int, payload: bytes) -> bytes:
    return struct.pack("<IB", 1 + len(payload), tag) + payload


def hello(v=1):
    return frame(TAGS["hello"], struct.pack("<I", v))


def model_digest(structure: bytes, weights: bytes, c: float) -> bytes:
    return hashlib.sha256(structure + weights + struct.pack("<d", c)).digest()


def model_check(digest: bytes):
    return frame(TAGS["model_check"], digest)


def model_upload(structure: bytes, weights: bytes, c: float, name=b"m", digest=None):
    digest = digest or model_digest(structure, weights, c)
    p = digest + struct.pack("<d", c) + struct.pack("<I", len(name)) + name + struct.pack("<I", len(structure))
    p += structure + struct.pack("<Q", len(weights)) + weights
    return frame(TAGS["model_upload"], p)


def frame_data(floats) -> bytes:
    import numpy as np
    a = np.ascontiguousarray(floats, dtype="<f4")
    return frame(TAGS["frame_data"], struct.pack("<I", a.size) + a.tobytes())


def resolution(w, h):
    return frame(TAGS["resolution"], struct.pack("<II", w, h))


def frame_size(n):
    return frame(TAGS["frame_size"], struct.pack("<I", n))


def error_msg(code, msg: bytes):
    return frame(TAGS["error"], struct.pack("<II", code, len(msg)) + msg)


class Peer:
    def __init__(self, port: int, timeout=20.0):
        self.s = socket.create_connection(("127.0.0.1", port), timeout=timeout)
        self.s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        self.buf = b""

    def send(self, data: bytes):
        self.s.sendall(data)

    def recv_msg(self):
        """(tag_name, payload) or None on EOF."""
        while len(self.buf) < 5:
            d = self.s.recv(1 << 20)
            if not d:
                return None
            self.buf += d
        ln, tag = struct.unpack("<IB", self.buf[:5])
        while len(self.buf) < 4 + ln:
            d = self.s.recv(1 << 22)
            if not d:
                return None
            self.buf += d
        payload = self.buf[5:4 + ln]
        self.buf = self.buf[4 + ln:]
        return NAMES.get(tag, tag), payload

    def expect_error(self):
        m = self.recv_msg()
        assert m is not None and m[0] == "error", m
        code, ln = struct.unpack("<II", m[1][:8])
        return code, m[1][8:8 + ln].decode()

    def closed(self) -> bool:
        try:
            return self.recv_msg() is None
        except (ConnectionResetError, socket.timeout):
            return True

    def handshake(self):
        self.send(hello())
        m = self.recv_msg()
        assert m == ("hello_ack", struct.pack("<I", 1)), m

    def close(self):
        self.s.close()


def forward_result(payload: bytes):
    import numpy as np
    compute_s, k = struct.unpack("<dI", payload[:12])
    return compute_s, np.frombuffer(payload[12:], dtype="<f4", count=k)


class ServerProc:
    """Start a server binary that prints `listening on HOST:PORT (...)`, stop it by PID."""

    def __init__(self, argv, timeout=120.0):
        self.p = subprocess.Popen(argv, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
        t0 = time.time()
        line = ""
        while time.time() - t0 < timeout:
            line = self.p.stdout.readline()
            if line.startswith("listening on") or not line:
                break
        if not line.startswith("listening on"):
            self.p.kill()
            raise RuntimeError(f"server did not start: {line!r} {self.p.stderr.read()[-2000:]}")
        self.banner = line.strip()
        self.port = int(line.split()[2].split(":")[1])
        self.endpoint = f"127.0.0.1:{self.port}"

    def stop(self) -> str:
        if self.p.poll() is None:
            self.p.terminate()  # SIGTERM -> drain (server_main.cpp:48-80)
        try:
            out, _ = self.p.communicate(timeout=60)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        return out
