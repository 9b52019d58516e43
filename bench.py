"""Benchmark: OpenPose frames/sec through the AVEC destination path on B200.

Workload (BASELINE.json configs[1], "C2"): OpenPose COCO pose net, 656x368
frames, batch 8 per GPU — one FrameData of 8 frames folded into 24 channels,
exactly what the wire carries (proj/src/server.cpp:294-302). Random-init
weights (deterministic He-uniform, seed 1), synthetic frames from the
reference's frame generator (seed 7). A step = one forward cycle of 8 frames.

  value : frames/s with inputs resident in HBM (avec_forward_device), whole
          job, over the driver's --steps; `steady_state` repeats it over 200
          steps
  e2e   : frames/s through the reference-facing C-ABI call avec_forward with
          pinned HOST buffers — H2D of the frames and D2H of the heatmaps are
          inside the timed region every step (fixed: one host thread per slot)
  wire  : C2 through bin/avec-server over TCP loopback (native clients)
  roofline : tcgen05 conv kernel with the largest share of the step,
          algorithmic FLOPs of its launches / their CUDA-event durations (op by
          op, so against the BURST bf16 peak), plus the whole step's TFLOP/s
  cpu_baseline : the reference's own server path (oracle/_ref/ref_arm), rank 0,
          with as many concurrent reference sessions as the host has threads
          (up to 16; its MockPose backend is one FIFO thread by design)

The other BASELINE configs ride in the same line (rank 0, N = 1 unless noted):
  c1            configs[0]: 368x368 batch 1 through avec-server, driven by the
                UNMODIFIED reference client (oracle/_ref/ref_client): fps and
                per-cycle latency p50/p90, plus the device-only forward latency
  mockpose_wire the reference arm's own workload (MockPose segment means, C2
                shape, reference Session client, oracle/_ref/ref_arm) pointed
                at avec-server: the like-for-like server ratio
  c3_memcpy     configs[2]: forwarded H2D/D2H sweep 4 KB..256 MB (c = 1)
                through avec-server and through avec_forward
  c4            configs[3]: 8 concurrent client sessions on one avec-server
                over all N GPUs, one session per GPU placement (every N)
  c5            configs[4]: BODY_25 1312x736 batch 32, frame groups sharded
                over the N ranks (strong scaling; every N)

`--impl reference` runs the reference's CPU implementation of the path
(Server + MockPoseBackend + Session over TCP loopback, built from the
reference sources into oracle/_ref) on the same workload shape.

Multi-GPU (torchrun): one process per GPU, each runs its own frame groups
(frames are independent: no data-path collective); barrier + max-over-ranks
device time; value = all ranks' frames / max time ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "OpenPose frames/sec through AVEC server at 1/2/4/8 B200; conv tensor-pipe %"
# BASELINE.json configs[1] (C2, default) and configs[4] (C5)
CONFIGS = {
    "c2": dict(family="openpose_coco", divisor=192.0 / 57.0, width=656, height=368, global_batch=8,
               per_gpu_batch=True, scaling="weak",
               workload="C2: OpenPose COCO pose net, 656x368 frames, batch 8 per GPU"),
    "c5": dict(family="openpose_body25", divisor=192.0 / 78.0, width=1312, height=736, global_batch=32,
               per_gpu_batch=False, scaling="strong",
               workload="C5: OpenPose BODY_25 1312x736, batch 32 sharded across the GPUs"),
}
CFG = CONFIGS["c2"]
W, H, BATCH = CFG["width"], CFG["height"], CFG["global_batch"]  # BATCH = frames per rank per step
# Execution slots per GPU = cycles in flight. Measured (tools/ab_slots.sh):
# device-resident throughput saturates at 2 streams; the e2e C-ABI path gains
# from third and fourth slots (their H2D/D2H overlap the other cycles'
# kernels: 2 -> 3 -> 4 slots C2 2525 -> 2611 -> 2623, C5 840 -> 870 -> 889);
# through the wire 2 server slots beat 3-4 (host-side TCP work per extra
# concurrent cycle). AVEC_SLOTS / AVEC_WIRE_SLOTS override.
SLOTS = int(os.environ.get("AVEC_SLOTS", "4"))          # avec_ctx slots (e2e threads up to this)
DEV_STREAMS = 2                                        # cycles in flight for the device-resident value
WIRE_SLOTS = int(os.environ.get("AVEC_WIRE_SLOTS", "2"))


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(bf16=d["bf16_tflops"], bf16_sust=d["bf16_tflops_sustained"], hbm=d["hbm_gbs"],
                    src="measured")
    return dict(bf16=1590.0, bf16_sust=1400.0, hbm=6650.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.samples, self._stop = device, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def run_reference_arm(steps: int, warmup: int, width=None, height=None, batch=None, clients=1,
                      divisor=None) -> dict:
    width, height = width or W, height or H
    batch = batch or CFG["global_batch"]
    divisor = divisor or CFG["divisor"]
    exe = ROOT / "oracle" / "_ref" / "ref_arm"
    if not exe.exists():
        return {"ok": False, "error": f"{exe} not built"}
    out = subprocess.run([str(exe), "--width", str(width), "--height", str(height), "--batch", str(batch),
                          "--steps", str(steps), "--warmup", str(warmup), "--clients", str(clients),
                          "--divisor", repr(divisor)],
                         capture_output=True, text=True, timeout=1800)
    try:
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return {"ok": False, "error": (out.stdout + out.stderr)[-300:]}


def reference_clients() -> int:
    """Concurrent reference sessions for the reference arm: its MockPose backend
    is one FIFO thread by design (proj/src/server.cpp:84-111), so more sessions
    overlap the others' socket traffic with it until the backend is the bound.
    Measured on a 16-thread B200 host at C2 (8x656x368 cycles): 1 / 2 / 4 / 8 /
    16 sessions = 248 / 462 / 878 / 940 / 985 frames/s, the backend alone ~1025
    (7.8 ms per cycle). All the host threads it can use: up to 16 sessions."""
    return max(1, min(16, os.cpu_count() or 1))


def reference_main(args, rank: int, world: int) -> int:
    if rank != 0:
        return 0
    clients = reference_clients()
    r = run_reference_arm(args.steps, args.warmup, clients=clients)
    if not r.get("ok"):
        print(json.dumps({"impl": "reference", "unavailable": r.get("error", "ref_arm failed")}))
        return 0
    fps = r["fps"]
    gb = CFG["global_batch"]
    sample = (f"reference accelfwd Server+MockPoseBackend, {clients} concurrent Session clients over TCP loopback, "
              f"{args.steps} cycles each of {gb}x{W}x{H} frames (reference emulates OpenPose with segment means)")
    cores = min(os.cpu_count() or 1, 2 * clients + 1)  # a client and a session thread each, plus the dispatcher
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_cycle"],
        "higher_is_better": True, "scaling": CFG["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference harness gen_frame, seed 7)",
        "config": {"workload": CFG["workload"] + " (reference path: MockPose segment means)",
                   "global_batch": gb,
                   "parallelism": f"cpu, {clients} sessions over the reference server's FIFO backend thread"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_posenet_oracle_sample() -> dict:
    """Bounded sample of the CPU pose-net oracle: one 7x7 stage conv (Mconv2,
    128->128) on one 656x368 frame at the /8 level; extrapolated to frames/s via
    the net's total FLOPs. Test-infrastructure oracle, timed as the 'port' baseline."""
    import numpy as np
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    from paper_2103_04930_b200 import netspec
    rng = np.random.default_rng(0)
    x = O.bf16_round(rng.standard_normal((1, H // 8, W // 8, 128)).astype(np.float32))
    w = rng.standard_normal((128, 128, 7, 7)).astype(np.float32) * 0.02
    b = np.zeros(128, np.float32)
    t0 = time.perf_counter()
    O.conv2d_nhwc(x, w, b, relu=True, round_bf16=True)
    dt = time.perf_counter() - t0
    fl = 2.0 * (H // 8) * (W // 8) * 128 * 128 * 49
    per_frame = netspec.flops_per_frame(netspec.layers_for(CFG["family"]), H, W)
    return {"gflops": fl / dt / 1e9, "fps_extrapolated": (fl / dt) / per_frame,
            "cores": O.lib().oracle_threads(), "seconds": dt}


SERVER_BIN = ROOT / "paper_2103_04930_b200" / "bin" / "avec-server"
LOADGEN_BIN = ROOT / "paper_2103_04930_b200" / "bin" / "avec-loadgen"
REF_CLIENT = ROOT / "oracle" / "_ref" / "ref_client"
REF_ARM = ROOT / "oracle" / "_ref" / "ref_arm"


class AvecServer:
    """bin/avec-server as a subprocess; stopped by its own PID (SIGTERM drain)."""

    def __init__(self, devices: str, slots: int, policy: str = "affinity"):
        self.p = subprocess.Popen([str(SERVER_BIN), "--devices", devices, "--slots", str(slots), "--policy", policy],
                                  stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
        line = self.p.stdout.readline()
        if not line.startswith("listening on"):
            err = self.p.stderr.read()[-300:]
            self.p.kill()
            raise RuntimeError("avec-server did not start: " + line + err)
        self.endpoint = line.split()[2]

    def close(self):
        self.p.terminate()
        try:
            self.p.wait(timeout=60)
        except subprocess.TimeoutExpired:
            self.p.kill()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _json_tail(out: str) -> dict:
    return json.loads(out.strip().splitlines()[-1])


def loadgen(endpoint: str, clients: int, steps: int, batch: int, width: int, height: int, model: str,
            warmup: int = 2, elems: int = 0) -> dict:
    cmd = [str(LOADGEN_BIN), "--endpoint", endpoint, "--clients", str(clients), "--steps", str(steps),
           "--warmup", str(warmup), "--batch", str(batch), "--width", str(width), "--height", str(height),
           "--model", model]
    if elems:
        cmd += ["--elems", str(elems)]
    return _json_tail(subprocess.run(cmd, capture_output=True, text=True, timeout=900).stdout)


def wire_run(device: int, steps: int, clients: int, warmup: int = 2) -> dict:
    """C2 cycles through bin/avec-server (one GPU) from `clients` concurrent
    native sessions over TCP loopback (BASELINE "through AVEC server")."""
    try:
        with AvecServer(str(device), WIRE_SLOTS) as srv:
            model = "posenet-body25" if CFG["family"] == "openpose_body25" else "posenet"
            out = loadgen(srv.endpoint, clients, steps, BATCH, W, H, model, warmup=warmup)
            out["transport"] = f"TCP loopback, native client (bin/avec-loadgen), avec-server --slots {WIRE_SLOTS}"
            return out
    except Exception as e:  # noqa: BLE001
        return {"ok": False, "error": str(e)}


def c1_run(be, device: int) -> dict:
    """configs[0]: one 368x368 frame per cycle, COCO, through avec-server,
    driven by the unmodified reference client (accelfwd::client::Session)."""
    import numpy as np
    import torch
    from paper_2103_04930_b200 import Dims, make_model, netspec
    res = {"workload": "C1: COCO 368x368 batch 1 per cycle, reference client -> avec-server over TCP loopback"}
    try:
        import tempfile
        spec = pathlib.Path(tempfile.mkdtemp()) / "coco.spec"
        spec.write_bytes(netspec.spec())
        with AvecServer(str(device), 2) as srv:
            r = subprocess.run([str(REF_CLIENT), "--endpoint", srv.endpoint, "--structure", str(spec),
                                "--name", "openpose_coco", "--divisor", repr(netspec.COCO_DIVISOR),
                                "--width", "368", "--height", "368", "--batch", "1", "--frames", "200",
                                "--warmup", "10"], capture_output=True, text=True, timeout=600)
            o = _json_tail(r.stdout)
        res.update({k: o.get(k) for k in ("ok", "fps", "lat_ms_p50", "lat_ms_p90", "lat_ms_max", "gpu_s_mean",
                                          "comm_s_mean", "byte_account_bad")})
        res["unit"] = "frames/s"
        # device-only latency of one frame: synchronous forward on resident input
        h = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
        dims = Dims(1, 3, 368, 368)
        x = torch.from_numpy(np.random.default_rng(1).random(dims.elem_count(), dtype=np.float32)).cuda(device)
        y = torch.empty(be.output_elems(h, dims), dtype=torch.float32, device=f"cuda:{device}")
        st = torch.cuda.Stream(device=device)
        lat = []
        for i in range(60):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            be.forward_device(h, dims, x.data_ptr(), y.data_ptr(), st.cuda_stream)
            e1.record(st)
            e1.synchronize()
            if i >= 10:
                lat.append(e0.elapsed_time(e1))
        lat.sort()
        res["device_ms_p50"] = round(lat[len(lat) // 2], 4)
        res["device_fps"] = round(1e3 / lat[len(lat) // 2], 1)
    except Exception as e:  # noqa: BLE001
        res.update(ok=False, error=str(e))
    return res


def mockpose_wire_run(device: int) -> dict:
    """The reference arm's own workload and client (ref_arm: reference Session,
    synthetic MockPose model, C2 shape) against avec-server instead of the
    reference Server: the like-for-like ratio of the two servers."""
    try:
        clients = reference_clients()  # the same sessions as the reference arm
        with AvecServer(str(device), 2) as srv:
            r = subprocess.run([str(REF_ARM), "--endpoint", srv.endpoint, "--width", str(W), "--height", str(H),
                                "--batch", str(CONFIGS["c2"]["global_batch"]), "--steps", "30", "--warmup", "3",
                                "--clients", str(clients)],
                               capture_output=True, text=True, timeout=600)
            o = _json_tail(r.stdout)
        o["workload"] = (f"reference arm workload (MockPose, 8x656x368 per cycle, {clients} reference Session "
                         f"clients) on avec-server")
        o["unit"] = "frames/s"
        return o
    except Exception as e:  # noqa: BLE001
        return {"ok": False, "error": str(e)}


def memcpy_sweep(be, device: int) -> dict:
    """configs[2]: forwarded H2D/D2H of 4 KB..256 MB per cycle. c = 1, so the
    reply is as large as the frame (MockPose with divisor 1 moves every byte
    both ways); GB/s counts in + out bytes per cycle."""
    import numpy as np
    from paper_2103_04930_b200 import Dims, Frame, PinnedBuffer, make_model
    sizes = [4 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]
    out = {"unit": "GB/s (in + out bytes per cycle)", "abi_pinned": [], "wire": []}
    try:
        h = be.register_model(make_model("memcpy", b"\x01\x02", b"", 1.0))
        for b in sizes:
            e = b // 4
            w = 4096 if e >= 4096 else e
            d = Dims(1, e // w, 1, w)
            pin_in, pin_out = PinnedBuffer(e), PinnedBuffer(e)
            pin_in.array[:] = np.random.default_rng(b).random(e, dtype=np.float32)
            fin = Frame(d, pin_in.array)
            reps = max(3, min(100, (256 << 20) // b))
            for _ in range(SLOTS):  # every execution slot sizes its device buffers once
                be.forward(h, fin, out=pin_out.array)
            t0 = time.perf_counter()
            for _ in range(reps):
                be.forward(h, fin, out=pin_out.array)
            dt = (time.perf_counter() - t0) / reps
            ok = bool(np.array_equal(pin_out.array, pin_in.array))
            out["abi_pinned"].append({"bytes": b, "us": round(dt * 1e6, 1), "gbs": round(2 * b / dt / 1e9, 2),
                                      "exact": ok})
            pin_in.free()
            pin_out.free()
        with AvecServer(str(device), 2) as srv:
            for b in sizes:
                e = b // 4
                w = 4096 if e >= 4096 else e
                reps = max(3, min(60, (256 << 20) // b))
                o = loadgen(srv.endpoint, 1, reps, 1, w, 1, "mockpose-c1", elems=e)
                dt = o["wall_s"] / reps if o.get("ok") else None
                out["wire"].append({"bytes": b, "us": round(dt * 1e6, 1) if dt else None,
                                    "gbs": round(2 * b / dt / 1e9, 2) if dt else None})
        out["peak_wire_gbs"] = max((x["gbs"] or 0) for x in out["wire"])
    except Exception as e:  # noqa: BLE001
        out.update(ok=False, error=str(e))
    return out


def c4_run(rank: int, world: int, host_group) -> dict:
    """configs[3]: 8 concurrent client sessions on ONE avec-server spanning all
    N GPUs of the job, sessions pinned one per GPU (--policy session). Rank 0
    runs it while the other ranks wait at a host-side (gloo) barrier, so no
    NCCL kernel spins on the GPUs it uses."""
    import torch.distributed as dist
    res = None
    if world > 1:
        dist.barrier(group=host_group)
    if rank == 0:
        try:
            devs = ",".join(str(i) for i in range(world))
            with AvecServer(devs, 2, "session") as srv:
                o = loadgen(srv.endpoint, 8, 30, CONFIGS["c2"]["global_batch"], W, H, "posenet")
            res = {"ok": o.get("ok"), "fps": o.get("fps"), "clients": 8, "gpus": world, "unit": "frames/s",
                   "placement": "one avec-server over all GPUs, session k on GPU (k-1) mod N",
                   "cycle_ms": o.get("cycle_ms"), "gpu_ms": o.get("gpu_ms"),
                   "workload": "C4: 8 concurrent sessions of 8x656x368 COCO cycles"}
        except Exception as e:  # noqa: BLE001
            res = {"ok": False, "error": str(e)}
    if world > 1:
        dist.barrier(group=host_group)
    return res


def c5_run(args, rank: int, world: int, dev: int) -> dict:
    """configs[4]: BODY_25 1312x736, 32 frames per cycle sharded into frame
    groups over the ranks with the product partition (avec_frame_groups):
    device-resident frames/s (max over ranks), e2e through avec_forward with
    pinned host buffers, and the pixel-major conv kernel's roofline."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, PinnedBuffer, make_model, netspec
    from paper_2103_04930_b200.sharding import frame_groups
    cfg = CONFIGS["c5"]
    w5, h5, total = cfg["width"], cfg["height"], cfg["global_batch"]
    first, nb = frame_groups(total, world)[rank]
    T = 3  # host threads (and slots) for the e2e leg: the 370 MB H2D of one cycle overlaps the others' compute
    be = B200Backend(dev, slots=T)
    try:
        h = be.register_model(make_model(cfg["family"], netspec.spec(cfg["family"]), b"", cfg["divisor"]))
        dims = Dims(1, 3 * nb, h5, w5)
        E, K = dims.elem_count(), be.output_elems(h, dims)
        rng = np.random.default_rng(11 + rank)
        host = (rng.integers(0, 1 << 24, E, dtype=np.int64) * (1.0 / (1 << 24))).astype(np.float32)
        d_in = torch.from_numpy(host).to(f"cuda:{dev}")
        # one stream per slot: the context leases slots round-robin, so call i
        # lands on slot i % T and stream i % T; the warm-up builds every slot's
        # plan (a plan built inside the timed region cost up to 100 ms per step)
        d_out = [torch.empty(K, dtype=torch.float32, device=f"cuda:{dev}") for _ in range(T)]
        streams = [torch.cuda.Stream(device=dev) for _ in range(T)]
        steps = 2 * T
        for i in range(2 * T):
            be.forward_device(h, dims, d_in.data_ptr(), d_out[i % T].data_ptr(), streams[i % T].cuda_stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(streams[0])
        for st in streams[1:]:
            st.wait_event(ev0)
        for i in range(steps):
            be.forward_device(h, dims, d_in.data_ptr(), d_out[i % T].data_ptr(), streams[i % T].cuda_stream)
        for st in streams[1:]:
            evb = torch.cuda.Event()
            evb.record(st)
            streams[0].wait_event(evb)
        ev1.record(streams[0])
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        value = steps * total / (ms / 1e3)
        # e2e: pinned host in/out through avec_forward, T host threads (one per slot)
        pin_in, pin_out = [PinnedBuffer(E) for _ in range(T)], [PinnedBuffer(K) for _ in range(T)]
        for j in range(T):
            pin_in[j].array[:] = host
        frames = [Frame(dims, pin_in[j].array) for j in range(T)]
        warm = [threading.Thread(target=be.forward, args=(h, frames[j]), kwargs={"out": pin_out[j].array})
                for j in range(T)]
        for t in warm:  # concurrent: every slot builds its plan
            t.start()
        for t in warm:
            t.join()
        if world > 1:
            dist.barrier()

        def worker(j, n):
            for _ in range(n):
                be.forward(h, frames[j], out=pin_out[j].array)
                float(pin_out[j].array[0])

        # 4 cycles per thread: the first cycle's H2D and the last one's D2H
        # (no compute to hide behind) are ~10 ms each on a ~30 ms cycle
        n_cyc = 4
        t0 = time.perf_counter()
        th = [threading.Thread(target=worker, args=(j, n_cyc)) for j in range(T)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([s], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            s = float(t.item())
        e2e = n_cyc * T * total / s
        prof = be.profile(h, dims, d_in.data_ptr(), reps=1)
        pm = [p for p in prof if p["kind"] == "conv_pm"]
        pm_fl, pm_ms = sum(p["flops"] for p in pm), sum(p["ms"] for p in pm)
        peaks = load_peaks()
        net_fl = netspec.flops_per_frame(netspec.layers_for(cfg["family"]), h5, w5)
        tf = pm_fl / (pm_ms / 1e3) / 1e12
        res = {"value": round(value, 2), "unit": "frames/s", "ms_per_step": round(ms / steps, 3),
               "frames_per_step": total, "frames_per_gpu": nb, "steps": steps, "scaling": "strong",
               "e2e": {"value": round(e2e, 2), "unit": "frames/s", "h2d_bytes_per_step": E * 4 * world,
                       "d2h_bytes_per_step": K * 4 * world, "api": f"avec_forward, pinned host buffers, {T} threads",
                       "cycles": n_cyc * T},
               "roofline": {"kernel": "conv_pm_kernel (tcgen05 pixel-major conv, all launches)", "bound": "tensor",
                            "achieved": round(tf, 1), "unit": "TFLOP/s", "peak": peaks["bf16"],
                            "frac": round(tf / peaks["bf16"], 4), "peak_kind": "burst (op-by-op replay)",
                            "frac_of_sustained": round(tf / peaks["bf16_sust"], 4),
                            "share_of_step": round(pm_ms / sum(p["ms"] for p in prof), 4)},
               "step_tflops_per_gpu": round(nb * net_fl / (ms / steps / 1e3) / 1e12, 1),
               "workload": cfg["workload"]}
        for b in pin_in + pin_out:
            b.free()
        return res
    finally:
        be.close()


def ours_main(args, rank: int, world: int, local_rank: int) -> int:
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT / "tests"))
    from paper_2103_04930_b200 import B200Backend, Dims, PinnedBuffer, make_model, netspec

    dev = local_rank
    torch.cuda.set_device(dev)
    S = DEV_STREAMS
    be = B200Backend(dev, slots=SLOTS)
    model = make_model(CFG["family"], netspec.spec(CFG["family"]), b"", CFG["divisor"])
    h = be.register_model(model)
    dims = Dims(1, 3 * BATCH, H, W)
    E, K = dims.elem_count(), be.output_elems(h, dims)
    host_group = dist.new_group(backend="gloo") if world > 1 else None

    # synthetic frames with the harness's value distribution (U[0,1) on a 2^-24
    # grid, harness.cpp:29-42), distinct per rank and per rotating input buffer
    # so consecutive steps never reuse an input
    n_rot = 4
    rng = np.random.default_rng(7 + 1000 * rank)
    host_frames = [(rng.integers(0, 1 << 24, E, dtype=np.int64) * (1.0 / (1 << 24))).astype(np.float32)
                   for _ in range(n_rot)]
    d_in = [torch.from_numpy(f).to(f"cuda:{dev}") for f in host_frames]
    d_out = [torch.empty(K, dtype=torch.float32, device=f"cuda:{dev}") for _ in range(S)]
    # S cycles in flight, like the server's S execution slots per GPU
    streams = [torch.cuda.Stream(device=dev) for _ in range(S)]

    if world > 1:
        dist.barrier()

    # ---------------- device-resident throughput (value) ----------------
    def step(i):
        be.forward_device(h, dims, d_in[i % n_rot].data_ptr(), d_out[i % S].data_ptr(),
                          streams[i % S].cuda_stream)

    def timed(n_steps: int, clocks=None):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(streams[0])
        for st in streams[1:]:
            st.wait_event(ev0)
        for i in range(n_steps):
            step(i)
        for st in streams[1:]:
            ev_b = torch.cuda.Event()
            ev_b.record(st)
            streams[0].wait_event(ev_b)
        ev1.record(streams[0])
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms

    # at least one warm-up call per slot: the context leases slots round-robin
    # and a slot builds its plan on first use (never inside the timed region)
    for i in range(max(args.warmup, SLOTS)):
        step(i)
    with ClockSampler(dev) as clocks:
        dev_ms = timed(args.steps)
    torch.cuda.synchronize()
    frames_total = args.steps * BATCH * world
    value = frames_total / (dev_ms / 1e3)
    # the same measurement over >= 200 steps (steady state, clocks sampled again)
    ss_steps = max(200, args.steps)
    with ClockSampler(dev) as ss_clocks:
        ss_ms = timed(ss_steps)
    steady = {"steps": ss_steps, "value": round(ss_steps * BATCH * world / (ss_ms / 1e3), 2), "unit": "frames/s",
              "ms_per_step": round(ss_ms / ss_steps, 4), "clocks": ss_clocks.summary()}

    # ---------------- e2e through avec_forward with pinned host buffers ----------------
    T = SLOTS  # one host thread per execution slot (fixed, not a best-of)
    pin_in = [PinnedBuffer(E) for _ in range(T)]
    pin_out = [PinnedBuffer(K) for _ in range(T)]
    for j in range(T):
        pin_in[j].array[:] = host_frames[j % n_rot]
    from paper_2103_04930_b200 import Frame
    frames = [Frame(dims, pin_in[j].array) for j in range(T)]
    warm = [threading.Thread(target=be.forward, args=(h, frames[j]), kwargs={"out": pin_out[j].array})
            for j in range(T)]
    for t in warm:  # concurrent, so every slot builds its plan
        t.start()
    for t in warm:
        t.join()
    checksum = [0.0] * T

    def worker(j, n):
        s = 0.0
        for _ in range(n):
            be.forward(h, frames[j], out=pin_out[j].array)
            s += float(pin_out[j].array[0])  # host read of the step's result
        checksum[j] = s

    e2e_cycles = max(args.steps, 64)

    def e2e_run(threads: int) -> float:
        if world > 1:
            dist.barrier()
        counts = [e2e_cycles // threads + (1 if i < e2e_cycles % threads else 0) for i in range(threads)]
        t0 = time.perf_counter()
        ths = [threading.Thread(target=worker, args=(j, counts[j])) for j in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([s], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            s = float(t.item())
        return e2e_cycles * BATCH * world / s

    e2e = e2e_run(T)
    e2e_serial = e2e_run(1)  # one synchronous cycle at a time (latency-bound)

    # ---------------- through the wire: avec-server + native clients over TCP ----------------
    # 4 sessions per GPU: two cycles compute in the server's two slots while the
    # other two sessions stream their frames in / results out (measured sweep:
    # 1 -> 860, 2 -> 1324, 4 -> 2092, 8 -> 1990 fps on C2, profiles/README.md)
    wire = wire_run(dev, steps=max(20, args.steps // 4), clients=4)
    # one session: its repeat cycles are pipelined once a helper thread has
    # prepared the frame-group plans, so it gets more warm-up cycles
    wire1 = wire_run(dev, steps=max(30, args.steps // 4), clients=1, warmup=6)
    wire["one_session"] = {k: wire1.get(k) for k in ("ok", "fps", "cycle_ms", "comm_ms", "gpu_ms")}
    if world > 1:
        t = torch.tensor([wire.get("fps", 0.0) or 0.0], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        wire["fps_all_ranks"] = float(t.item())

    # ---------------- roofline of the dominant kernel ----------------
    prof = be.profile(h, dims, d_in[0].data_ptr(), reps=3)
    peaks = load_peaks()
    step_ms_prof = sum(p["ms"] for p in prof)
    # dominant kernel = the conv variant with the largest share of the step:
    # COCO: the swap-AB 7x7 stage conv (conv_tc_kernel<2>); BODY_25: pixel-major
    share = {k: sum(p["ms"] for p in prof if p["kind"] == k) for k in ("conv_tc", "conv_pm")}
    dom_kind = max(share, key=share.get)
    dom = [p for p in prof if p["kind"] == dom_kind]
    dom_fl = sum(p["flops"] for p in dom) / max(len(dom), 1)   # per launch
    dom_ms = sum(p["ms"] for p in dom) / max(len(dom), 1)      # mean launch duration
    dom_tf = dom_fl / (dom_ms / 1e3) / 1e12
    allc = [p for p in prof if p["kind"] in ("conv_tc", "conv_pm", "conv_first", "conv_head", "conv12")]  # every conv launch
    all_fl, all_ms = sum(p["flops"] for p in allc), sum(p["ms"] for p in allc)
    traffic = None
    tp = ROOT / "profiles" / "conv_traffic.json"
    if tp.exists() and args.config == "c2":  # ncu capture of the C2 dominant kernel
        try:
            traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")
        except Exception:
            pass
    net_fl = netspec.flops_per_frame(netspec.layers_for(CFG["family"]), H, W)
    kernel_name = {"conv_tc": "conv_tc_kernel<2>: tcgen05 swap-AB 7x7 stage conv (L1+L2 branch pair per launch)",
                   "conv_pm": "conv_pm_kernel<N,S>: tcgen05 pixel-major conv (all launches of the class)"}
    step_tf = BATCH * net_fl / (dev_ms / args.steps / 1e3) / 1e12
    ss_tf = BATCH * net_fl / (ss_ms / ss_steps / 1e3) / 1e12
    roofline = {
        "bound": "tensor",
        "kernel": kernel_name[dom_kind],
        "achieved": round(dom_tf, 1), "peak": peaks["bf16"], "unit": "TFLOP/s",
        "frac": round(dom_tf / peaks["bf16"], 4), "traffic": traffic,
        "peak_kind": f"{peaks['src']} burst bf16: kernels timed op by op in isolation (avec_posenet_profile)",
        "frac_of_sustained": round(dom_tf / peaks["bf16_sust"], 4),
        "flops_per_launch": dom_fl, "launch_ms": round(dom_ms, 4), "launches_per_step": len(dom),
        "share_of_step": round(sum(p["ms"] for p in dom) / step_ms_prof, 4),
        "all_conv": {"achieved": round(all_fl / (all_ms / 1e3) / 1e12, 1),
                     "frac": round(all_fl / (all_ms / 1e3) / 1e12 / peaks["bf16"], 4),
                     "launches_per_step": len(allc), "share_of_step": round(all_ms / step_ms_prof, 4)},
        "net_flops_per_frame": net_fl,
        "step": {"tflops_per_gpu": round(step_tf, 1), "frac_burst": round(step_tf / peaks["bf16"], 4),
                 "frac_sustained": round(step_tf / peaks["bf16_sust"], 4),
                 "steady_tflops_per_gpu": round(ss_tf, 1), "steady_frac_burst": round(ss_tf / peaks["bf16"], 4),
                 "steady_frac_sustained": round(ss_tf / peaks["bf16_sust"], 4)},
    }
    breakdown = {}
    for p in prof:
        k = p["kind"]
        breakdown.setdefault(k, {"ms": 0.0, "launches": 0})
        breakdown[k]["ms"] = round(breakdown[k]["ms"] + p["ms"], 4)
        breakdown[k]["launches"] += 1
    for b in pin_in + pin_out:
        b.free()

    # ---------------- the other BASELINE configs ----------------
    extras = {}
    if args.config == "c2":
        if world == 1:
            extras["c1"] = c1_run(be, dev)
            extras["mockpose_wire"] = mockpose_wire_run(dev)
            extras["c3_memcpy"] = memcpy_sweep(be, dev)
        be.close()
        be = None
        torch.cuda.synchronize()
        extras["c4"] = c4_run(rank, world, host_group)
        try:
            extras["c5"] = c5_run(args, rank, world, dev)
        except Exception as e:  # noqa: BLE001
            extras["c5"] = {"ok": False, "error": str(e)}

    if rank == 0:
        ref_cycles = 30 if args.config == "c2" else 3  # per session; a few seconds of reference CPU work
        ref_clients = reference_clients() if args.config == "c2" else 1
        ref = (run_reference_arm(steps=ref_cycles, warmup=1, clients=ref_clients) if world == 1
               else {"ok": False, "error": "rank0 N>1"})
        try:
            port = cpu_posenet_oracle_sample() if world == 1 else None
        except Exception as e:  # noqa: BLE001
            port = {"error": str(e)}
        cpu = None
        if ref.get("ok"):
            cpu = {"value": ref["fps"], "unit": "frames/s", "cores": min(os.cpu_count() or 1, 2 * ref_clients + 1),
                   "kind": "reference",
                   "sample": f"reference Server+MockPoseBackend, {ref_clients} concurrent Session client(s) over TCP "
                             f"loopback, {ref_cycles} cycles each of {CFG['global_batch']}x{W}x{H} (the reference "
                             f"emulates OpenPose with segment means)",
                   "posenet_oracle_port": port}
            mw = extras.get("mockpose_wire")
            if mw and mw.get("ok"):
                mw["reference_server_fps"] = ref["fps"]
                mw["ratio_vs_reference_server"] = round(mw["fps"] / ref["fps"], 2)
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 4),
            "higher_is_better": True, "scaling": CFG["scaling"], "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic frames (harness distribution U[0,1) on a 2^-24 grid), random-init He-uniform "
                    "weights (seed 1)",
            "config": {"workload": CFG["workload"], "family": CFG["family"],
                       "global_batch": BATCH * world, "frame": f"{W}x{H}", "frames_per_gpu": BATCH,
                       "parallelism": f"frame groups x{world}",
                       "l2": "4 rotating input buffers; per-step activation working set >> 126 MB L2"},
            "steady_state": steady,
            "e2e": {"value": round(e2e, 2), "unit": "frames/s", "h2d_bytes_per_step": E * 4,
                    "d2h_bytes_per_step": K * 4, "cycles": e2e_cycles,
                    "api": f"avec_forward (pinned host buffers), {T} host threads over {SLOTS} slots",
                    "one_thread": round(e2e_serial, 2)},
            "wire": wire,
            "roofline": roofline, "cpu_baseline": cpu,
            "gpu_launches": args.steps * len(prof),
            "clocks": clocks.summary(),
            "kernel_breakdown_ms_per_step": breakdown,
        }
        if world == 1 and args.config == "c2":
            # the reference's own server path (Server + MockPoseBackend on one
            # host thread, reference Session clients, TCP loopback) on each
            # config's shape, beside our number
            legs = {"c1": dict(width=368, height=368, batch=1, steps=200, warmup=5),
                    "c4": dict(width=W, height=H, batch=8, steps=8, warmup=1, clients=8),
                    "c5": dict(width=CONFIGS["c5"]["width"], height=CONFIGS["c5"]["height"],
                               batch=CONFIGS["c5"]["global_batch"], steps=2, warmup=1,
                               divisor=CONFIGS["c5"]["divisor"])}
            for key, kw in legs.items():
                if isinstance(extras.get(key), dict):
                    r = run_reference_arm(**kw)
                    extras[key]["reference_cpu"] = {
                        "ok": r.get("ok"), "fps": r.get("fps"), "unit": "frames/s", "cores": 1,
                        "kind": "reference", "error": r.get("error"),
                        "sample": f"reference Server+MockPoseBackend, {kw.get('clients', 1)} Session client(s) over "
                                  f"TCP loopback, {kw['steps']} cycles of {kw['batch']}x{kw['width']}x{kw['height']}"}
        line.update(extras)
        print(json.dumps(line))
    if be is not None:
        be.close()
    return 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    global CFG, W, H, BATCH
    CFG = CONFIGS[args.config]
    W, H = CFG["width"], CFG["height"]
    if CFG["per_gpu_batch"]:
        BATCH = CFG["global_batch"]  # weak scaling: every GPU runs its own batch
    else:
        if CFG["global_batch"] % world:
            raise SystemExit(f"{args.config}: global batch {CFG['global_batch']} does not split over {world} GPUs")
        BATCH = CFG["global_batch"] // world  # strong scaling: one batch sharded into frame groups
    if args.config == "c5" and args.steps == 200:
        args.steps = 20  # 32 frames of 1312x736 per step: keep the default run within minutes
    if args.impl == "reference":
        return reference_main(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        # NCCL prints its version banner to stdout at NCCL_DEBUG=VERSION or WARN;
        # keep rank 0's stdout one JSON line (unset = no banner)
        if os.environ.get("NCCL_DEBUG", "").upper() in ("VERSION", "WARN"):
            os.environ["NCCL_DEBUG"] = "NONE"
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    try:
        return ours_main(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
