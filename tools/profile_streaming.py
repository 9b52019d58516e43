"""Run the streaming (HBM-bound) kernels once each at BASELINE sizes, for ncu
captures of their achieved DRAM bandwidth (north star: "achieved HBM GB/s for
the streaming layers"):
  * segmean (MockPose, the reference's model) on a C2 (8x656x368) and a C5
    (32x1312x736) FrameData, device-resident;
  * x8 bilinear upsample of the C2 net output (8 x 57 planes of 46x82);
  * 3x3 peak NMS on the 8 x 18 upsampled body-part heatmaps;
  * the fused x8 upsample + NMS on those 144 planes (checked identical to the pair);
  * the pose net's remaining max-pool (one C2 forward).

    ncu --set full -k regex:'segmean|upsample|nms|maxpool' python tools/profile_streaming.py
"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch
    from paper_2103_04930_b200 import B200Backend, Dims, make_model, netspec
    be = B200Backend(0, slots=1)
    rng = np.random.default_rng(7)
    # MockPose (opaque structure -> segment means), c = 192/57
    hm = be.register_model(make_model("pose-est", bytes(range(16)), b"\x01", 192.0 / 57.0))
    for (n, w, h) in ((8, 656, 368), (32, 1312, 736)):
        dims = Dims(1, 3 * n, h, w)
        x = torch.from_numpy(rng.random(dims.elem_count(), dtype=np.float32)).cuda()
        y = torch.empty(be.output_elems(hm, dims), dtype=torch.float32, device="cuda")
        be.forward_device(hm, dims, x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
    # pose net C2: forward (max-pool inside), then upsample + NMS on its output
    hp = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    dims = Dims(1, 24, 368, 656)
    x = torch.from_numpy(rng.random(dims.elem_count(), dtype=np.float32)).cuda()
    out = torch.empty(be.output_elems(hp, dims), dtype=torch.float32, device="cuda")
    be.forward_device(hp, dims, x.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    planes = 8 * 57
    up = torch.empty((planes, 368, 656), dtype=torch.float32, device="cuda")
    be.upsample_device(out.data_ptr(), planes, 46, 82, 8, up.data_ptr())
    heat = up.view(8, 57, 368, 656)[:, :18].contiguous().view(-1, 368, 656)
    maxp = 128
    cnt = torch.zeros(heat.shape[0], dtype=torch.int32, device="cuda")
    pk = torch.zeros((heat.shape[0], maxp, 5), dtype=torch.float32, device="cuda")
    # two thresholds: the median (a many-peak stress case: most warp rows hold
    # peaks) and the 99.9th percentile (sparse peaks, as on real heatmaps)
    sample = heat[0].flatten()[::97]
    for q in (0.5, 0.999):
        thr = float(torch.quantile(sample, q))
        be.nms_device(heat.data_ptr(), heat.shape[0], 368, 656, thr, maxp, cnt.data_ptr(), pk.data_ptr())
        torch.cuda.synchronize()
        print("ok", q, int(cnt.sum()))
    # the fused pair on the same 144 heatmap planes (upsample written once,
    # not read back), against the two launches it replaces
    src = out.view(8, 57, 46, 82)[:, :18].contiguous()
    up2 = torch.empty((144, 368, 656), dtype=torch.float32, device="cuda")
    cnt2 = torch.zeros_like(cnt)
    pk2 = torch.zeros_like(pk)
    for q in (0.5, 0.999):
        thr = float(torch.quantile(sample, q))
        be.upsample_nms_device(src.data_ptr(), 144, 46, 82, 8, thr, maxp, up2.data_ptr(), cnt2.data_ptr(),
                               pk2.data_ptr())
        be.nms_device(heat.data_ptr(), 144, 368, 656, thr, maxp, cnt.data_ptr(), pk.data_ptr())
        torch.cuda.synchronize()
        same = torch.equal(up2, heat) and torch.equal(cnt2, cnt) and torch.equal(pk2, pk)
        print("fused ok", q, int(cnt2.sum()), "identical" if same else "DIFFERENT")
    if "--time" in sys.argv:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        thr = float(torch.quantile(sample, 0.5))
        for name, fn in (("split", lambda: (be.upsample_device(src.data_ptr(), 144, 46, 82, 8, up2.data_ptr()),
                                            be.nms_device(up2.data_ptr(), 144, 368, 656, thr, maxp,
                                                          cnt2.data_ptr(), pk2.data_ptr()))),
                         ("fused", lambda: be.upsample_nms_device(src.data_ptr(), 144, 46, 82, 8, thr, maxp,
                                                                  up2.data_ptr(), cnt2.data_ptr(), pk2.data_ptr()))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ev[0].record()
            for _ in range(20):
                fn()
            ev[1].record()
            torch.cuda.synchronize()
            print(name, "%.1f us per call (incl. the per-call host sync)" % (ev[0].elapsed_time(ev[1]) * 1e3 / 20))
    be.close()


if __name__ == "__main__":
    main()
