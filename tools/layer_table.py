"""Per-launch table of one pose-net forward (device timings via
avec_posenet_profile): kind, GFLOP, ms, TFLOP/s, share of the step.

    python tools/layer_table.py --config c5 [--json out.json]
"""
import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c5"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default="")
    ap.add_argument("--input", default="bf16", choices=["bf16", "tf32"], help="first-layer operand precision")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2103_04930_b200 import B200Backend, Dims, make_model, netspec
    fam, W, H, B, div = {
        "c1": ("openpose_coco", 368, 368, 1, netspec.COCO_DIVISOR),
        "c2": ("openpose_coco", 656, 368, 8, netspec.COCO_DIVISOR),
        "c5": ("openpose_body25", 1312, 736, 32, netspec.BODY25_DIVISOR),
    }[a.config]
    B = a.batch or B
    be = B200Backend(0, slots=1)
    h = be.register_model(make_model(fam, netspec.spec(fam, input_dtype=a.input), b"", div))
    dims = Dims(1, 3 * B, H, W)
    x = torch.from_numpy(np.random.default_rng(7).random(dims.elem_count(), dtype=np.float32)).cuda()
    prof = be.profile(h, dims, x.data_ptr(), reps=a.reps)
    total = sum(p["ms"] for p in prof)
    rows = []
    for i, p in enumerate(prof):
        tf = p["flops"] / (p["ms"] * 1e-3) / 1e12 if p["ms"] > 0 else 0.0
        gbs = p["bytes"] / (p["ms"] * 1e-3) / 1e9 if p["ms"] > 0 else 0.0
        rows.append(dict(i=i, kind=p["kind"], gflop=p["flops"] / 1e9, ms=p["ms"], tflops=tf, gbs=gbs,
                         share=p["ms"] / total))
        print(f"{i:3d} {p['kind']:13s} {p['flops'] / 1e9:9.1f} GF {p['ms'] * 1e3:8.1f} us "
              f"{tf:7.1f} TF/s {gbs:7.0f} GB/s {100 * p['ms'] / total:5.1f}%")
    conv_fl = sum(p["flops"] for p in prof)
    print(f"step {total:.3f} ms, {conv_fl / 1e12:.2f} TFLOP, {conv_fl / (total * 1e-3) / 1e12:.1f} TFLOP/s")
    by = {}
    for p in prof:
        k = by.setdefault(p["kind"], [0, 0.0, 0.0])
        k[0] += 1
        k[1] += p["ms"]
        k[2] += p["flops"]
    for k, (n, ms, fl) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:12s} {n:3d} launches {ms:8.3f} ms {100 * ms / total:5.1f}% "
              f"{fl / (ms * 1e-3) / 1e12 if ms else 0:7.1f} TF/s")
    if a.json:
        pathlib.Path(a.json).write_text(json.dumps(dict(config=a.config, batch=B, step_ms=total, rows=rows),
                                                   indent=1))
    be.close()


if __name__ == "__main__":
    main()
