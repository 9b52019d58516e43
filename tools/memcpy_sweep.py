"""C3: forwarded-memcpy sweep 4 KB .. 256 MB (BASELINE.json configs[2]).

Each size is one FrameData of E = bytes/4 floats answered with c = 1, so the
result is as large as the input (MockPose with divisor 1 is the identity on
the wire). Sizes go through
  * the C-ABI (avec_forward, pinned and pageable host buffers): H2D + D2H via
    the slot's pinned double-buffered staging, GB/s of (in + out) bytes;
  * the wire: avec-server over TCP loopback, driven by the native client.
Prints one JSON object; results for the round go to profiles/.
"""
import json
import pathlib
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import numpy as np
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, PinnedBuffer, make_model
    be = B200Backend(0, slots=2)
    h = be.register_model(make_model("memcpy", b"\x01\x02", b"", 1.0))
    sizes = [4 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]
    res = {"abi_pinned": [], "abi_pageable": [], "wire": []}
    for b in sizes:
        e = b // 4
        w = (4096 if e // 1024 > 65535 else 1024) if e % 1024 == 0 else e
        d = Dims(1, e // w, 1, w)
        src = np.random.default_rng(b).random(e, dtype=np.float32)
        reps = max(3, min(200, (256 << 20) // b))
        for kind in ("abi_pinned", "abi_pageable"):
            if kind == "abi_pinned":
                pin_in, pin_out = PinnedBuffer(e), PinnedBuffer(e)
                pin_in.array[:] = src
                fin, out = Frame(d, pin_in.array), pin_out.array
            else:
                fin, out = Frame(d, src), np.empty(e, np.float32)
            for _ in range(2):  # warm both execution slots (device buffers sized on first use)
                be.forward(h, fin, out=out)
            t0 = time.perf_counter()
            for _ in range(reps):
                be.forward(h, fin, out=out)
            dt = (time.perf_counter() - t0) / reps
            assert np.array_equal(out, src)
            res[kind].append({"bytes": b, "us": round(dt * 1e6, 1), "gbs_in_plus_out": round(2 * b / dt / 1e9, 2)})
    # wire: the native client against avec-server, same sizes
    srv = subprocess.Popen([str(ROOT / "paper_2103_04930_b200" / "bin" / "avec-server")], stdout=subprocess.PIPE,
                           text=True)
    line = srv.stdout.readline()
    ep = line.split()[2]
    try:
        for b in sizes:
            e = b // 4
            reps = max(3, min(100, (256 << 20) // b))
            w = 4096 if e // 1024 > 65535 else min(e, 1024)
            r = subprocess.run([str(ROOT / "paper_2103_04930_b200" / "bin" / "avec-loadgen"), "--endpoint", ep,
                                "--model", "mockpose-c1", "--clients", "1", "--steps", str(reps), "--warmup", "2",
                                "--batch", "1", "--width", str(w), "--height", "1",
                                "--elems", str(e)], capture_output=True, text=True, timeout=600)
            o = json.loads(r.stdout.strip().splitlines()[-1])
            dt = o["wall_s"] / reps if o.get("ok") else None
            res["wire"].append({"bytes": b, "us": round(dt * 1e6, 1) if dt else None,
                                "gbs_in_plus_out": round(2 * b / dt / 1e9, 2) if dt else None,
                                "error": o.get("error")})
    finally:
        srv.terminate()
        srv.wait(timeout=60)
    be.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
