"""Per-CTA timeline of one pixel-major conv launch (latency study).

Needs a trace build of libavec_cuda.so (-DAVEC_TRACE; tools/trace_op.sh makes
one in a scratch copy of the repo). Runs avec_posenet_profile on one shape
with AVEC_TRACE_OP=<op> and prints, per stamp, the min / median / max time
since the launch's first CTA started:
  0 CTA entry  1 prologue done  2 first window+weights issued  3 producer done
  4 MMA: first window landed  5 MMA: last tile committed  6 epilogue: acc ready
  7 epilogue: stores issued  8 epilogue: stores complete  9 CTA exit
    python tools/trace_op.py --config c1 --op 1
"""
import argparse
import ctypes
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--op", type=int, default=1)
    a = ap.parse_args()
    os.environ["AVEC_TRACE_OP"] = str(a.op)
    import numpy as np
    import torch
    from paper_2103_04930_b200 import B200Backend, Dims, _lib, make_model, netspec
    W, H, B = {"c1": (368, 368, 1), "c2": (656, 368, 8), "c2b1": (656, 368, 1)}[a.config]
    be = B200Backend(0, slots=1)
    h = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    dims = Dims(1, 3 * B, H, W)
    x = torch.from_numpy(np.random.default_rng(7).random(dims.elem_count(), dtype=np.float32)).cuda()
    prof = be.profile(h, dims, x.data_ptr(), reps=3)
    L = _lib.load()
    buf = (ctypes.c_ulonglong * (296 * 16))()
    dump = L.avec_trace_dump_tc if prof[a.op]["kind"] == "conv_tc" else L.avec_trace_dump
    assert dump(buf, 296 * 16) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(296, 16).astype(np.float64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    print(f"op {a.op} ({prof[a.op]['kind']}, {prof[a.op]['ms'] * 1e3:.1f} us in the profile), {used.sum()} CTAs")
    names = ["entry", "prologue", "1st load issued", "producer done", "1st window landed", "mma done",
             "acc ready (epi)", "stores issued", "stores done", "exit"]  # conv_tc: no 2, 3
    for k, n in enumerate(names):
        v = t[:, k]
        v = v[v > 0] - t0
        if v.size:
            print(f"  {k} {n:18s} min {v.min() / 1e3:7.2f}  med {np.median(v) / 1e3:7.2f}  max {v.max() / 1e3:7.2f} us")
    be.close()


if __name__ == "__main__":
    main()
