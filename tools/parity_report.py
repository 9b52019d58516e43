"""Per-layer parity numbers at the benchmarked shapes (the same checks as
tests/test_gpu_fullsize.py, recorded instead of asserted):

    python tools/parity_report.py --out profiles/r02_parity_fullsize.json

For every conv layer: relative L2 error and max |gpu - oracle| over the
sampled rows, the number of rows, and how the plan executes the layer."""
import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import fullsize as F
    import oracle_lib as O
    from paper_2103_04930_b200 import B200Backend, Dims, Frame, make_model, netspec, synth_posenet_weights
    shapes = [("c2", "openpose_coco", 656, 368, 8, 7, 2), ("coco_1312x736_b8", "openpose_coco", 1312, 736, 8, 9, 3),
              ("c5", "openpose_body25", 1312, 736, 32, 7, 5)]
    report = {}
    for name, fam, w, hgt, nb, seed, rseed in shapes:
        be = B200Backend(0, slots=1)
        s = netspec.spec(fam)
        div = netspec.BODY25_DIVISOR if fam == "openpose_body25" else netspec.COCO_DIVISOR
        h = be.register_model(make_model(fam, s, b"", div))
        layers = netspec.layers_for(fam)
        wb = [(O.bf16_round(x), b, sl) for x, b, sl in netspec.split_weights(layers, synth_posenet_weights(s))]
        frame = Frame(Dims(1, 3 * nb, hgt, w), O.batched_frame(w, hgt, nb, seed=seed))
        finals = ({"Mconv7_stage3_L2", "Mconv7_stage1_L1"} if fam == "openpose_body25"
                  else {"Mconv7_stage6_L1", "Mconv7_stage6_L2"})
        rows = []
        for i, L in enumerate(layers):
            kind, src = be.layer_fusion(h, frame.dims, i)
            r = F.check_layer_rows(be, h, frame, layers, wb, i, final=L.name in finals, seed=rseed)
            rows.append(dict(layer=L.name, fusion=kind, rel_err=r[0] if r else None,
                             max_abs=r[1] if r else None, rows=r[2] if r else 0))
        errs = [x["rel_err"] for x in rows if x["rel_err"] is not None]
        report[name] = dict(family=fam, frames=nb, width=w, height=hgt, layers_checked=len(errs),
                            worst_rel_err=max(errs), median_rel_err=sorted(errs)[len(errs) // 2], per_layer=rows)
        print(name, len(errs), "layers, worst", max(errs), flush=True)
        be.close()
    if a.out:
        pathlib.Path(a.out).write_text(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
