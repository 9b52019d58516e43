"""Run a pose-net forward a few times (for ncu captures): warm-up + `--iters` forwards.

    ncu --set full -k regex:conv_ -s <skip> -c <n> python tools/profile_forward.py
"""
import argparse
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--width", type=int, default=656)
    ap.add_argument("--height", type=int, default=368)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--family", default="openpose_coco", choices=["openpose_coco", "openpose_body25"])
    a = ap.parse_args()
    import numpy as np
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec
    import oracle_lib as O
    be = B200Backend(0, slots=1)
    div = netspec.COCO_DIVISOR if a.family == "openpose_coco" else netspec.BODY25_DIVISOR
    h = be.register_model(make_model(a.family, netspec.spec(a.family), b"", div))
    f = Frame(Dims(1, 3 * a.batch, a.height, a.width), O.batched_frame(a.width, a.height, a.batch))
    out = be.forward(h, f).data  # warm: builds the plan and graph
    for _ in range(a.iters):
        out = be.forward(h, f).data
    print("ok", out.size, float(np.abs(out).sum()))


if __name__ == "__main__":
    main()
