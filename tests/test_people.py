"""Bottom-up person assembly (SURVEY §8 f rank 4): PAF candidate scores on the
GPU bit-exact against oracle/paf_oracle.c, and the product's host assembly
(avec_assemble_people) identical to the oracle's."""
import numpy as np
import pytest

import oracle_lib as O

N_PARTS = 18


def synthetic_scene(H=96, W=128, people=2, seed=3):
    """Stick figures: keypoints per person, PAF planes painted with the limb's
    unit vector within 2 px of each limb segment, NMS-style peak arrays."""
    from paper_2103_04930_b200 import coco_limbs
    rng = np.random.default_rng(seed)
    parts, pafidx, new_rows = coco_limbs()
    max_peaks = 8
    kp = np.zeros((people, N_PARTS, 2), np.float32)
    for p in range(people):
        cx, cy = 30 + 60 * p, 20
        base = np.array([[0, 0], [0, 8], [-8, 8], [-12, 20], [-14, 32], [8, 8], [12, 20], [14, 32], [-5, 36],
                         [-6, 52], [-6, 68], [5, 36], [6, 52], [6, 68], [-2, -2], [2, -2], [-4, 0], [4, 0]],
                        np.float32)
        kp[p] = base + np.array([cx, cy], np.float32) + rng.integers(-1, 2, (N_PARTS, 2))
    counts = np.full(N_PARTS, people, np.int32)
    peaks = np.zeros((N_PARTS, max_peaks, 5), np.float32)
    for j in range(N_PARTS):
        for p in range(people):
            peaks[j, p, 0:2] = kp[p, j]
            peaks[j, p, 2:4] = kp[p, j]
            peaks[j, p, 4] = 0.6 + 0.1 * p
    paf = np.zeros((38, H, W), np.float32)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float32)
    for l in range(parts.shape[0]):
        for p in range(people):
            a, b = kp[p, parts[l, 0]], kp[p, parts[l, 1]]
            d = b - a
            n = float(np.hypot(*d))
            if n == 0:
                continue
            u = d / n
            t = np.clip(((xx - a[0]) * u[0] + (yy - a[1]) * u[1]) / n, 0, 1)
            dist = np.hypot(xx - (a[0] + t * d[0]), yy - (a[1] + t * d[1]))
            m = dist <= 2.0
            paf[pafidx[l, 0]][m] = u[0]
            paf[pafidx[l, 1]][m] = u[1]
    return paf, counts, peaks, parts, pafidx, new_rows


def test_assembly_matches_oracle_random_candidates():
    from paper_2103_04930_b200 import assemble_people, coco_limbs
    parts, _, new_rows = coco_limbs()
    rng = np.random.default_rng(5)
    max_peaks = 6
    for trial in range(20):
        counts = rng.integers(0, max_peaks + 1, N_PARTS).astype(np.int32)
        peaks = np.zeros((N_PARTS, max_peaks, 5), np.float32)
        peaks[:, :, 4] = rng.random((N_PARTS, max_peaks)).astype(np.float32)
        cand = np.zeros((parts.shape[0], max_peaks, max_peaks, 2), np.float32)
        cand[..., 0] = rng.random(cand.shape[:3]).astype(np.float32)
        cand[..., 1] = (rng.random(cand.shape[:3]) < 0.3).astype(np.float32)
        got_p, got_s = assemble_people(counts, peaks, cand, parts, new_rows)
        ref_p, ref_s = O.assemble_people(counts, peaks, cand, parts, new_rows)
        assert np.array_equal(got_p, ref_p), trial
        assert got_s.tobytes() == ref_s.tobytes(), trial


def test_synthetic_scene_assembles_two_people_cpu():
    from paper_2103_04930_b200 import assemble_people
    paf, counts, peaks, parts, pafidx, new_rows = synthetic_scene()
    cand = O.paf_candidates(paf, counts, peaks, parts, pafidx, 0.05)
    people, score = assemble_people(counts, peaks, cand, parts, new_rows)
    assert people.shape[0] == 2
    assert (people >= 0).all()  # every part of both people found
    assert sorted(people[:, 0].tolist()) == [0, 1]


@pytest.mark.gpu
def test_paf_candidates_gpu_bitexact_synthetic():
    import torch
    from paper_2103_04930_b200 import B200Backend
    paf, counts, peaks, parts, pafidx, _ = synthetic_scene()
    be = B200Backend(0)
    H, W = paf.shape[1:]
    max_peaks = peaks.shape[1]
    d_paf = torch.from_numpy(paf).cuda()
    d_cnt = torch.from_numpy(counts).cuda()
    d_pk = torch.from_numpy(peaks).cuda()
    d_cand = torch.zeros((parts.shape[0], max_peaks, max_peaks, 2), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    be.paf_candidates_device(d_paf.data_ptr(), H, W, d_cnt.data_ptr(), d_pk.data_ptr(), max_peaks, parts, pafidx,
                             0.05, d_cand.data_ptr())
    got = d_cand.cpu().numpy()
    ref = O.paf_candidates(paf, counts, peaks, parts, pafidx, 0.05)
    assert got.tobytes() == ref.tobytes()
    # nearly every true limb of both people is a valid candidate (a short face
    # limb can sample another limb's painted band); assembly still finds both
    assert got[..., 1].sum() >= 2 * parts.shape[0] - 2
    be.close()


@pytest.mark.gpu
def test_people_pipeline_on_net_output():
    """net (COCO, 368x368) -> x8 upsample -> NMS on the 18 part maps -> PAF
    candidates on the upsampled PAF planes -> assembly; GPU stages bit-exact
    against the oracle at every step, assembly identical."""
    import torch
    from paper_2103_04930_b200 import (B200Backend, Dims, Frame, assemble_people, coco_limbs, make_model,
                                       netspec)
    h = w = 368
    be = B200Backend(0)
    hd = be.register_model(make_model("openpose_coco", netspec.spec(), b"", netspec.COCO_DIVISOR))
    out = be.forward(hd, Frame(Dims(1, 3, h, w), O.batched_frame(w, h, 1, seed=7))).data.reshape(57, 46, 46)
    d_net = torch.from_numpy(np.ascontiguousarray(out)).cuda()
    d_up = torch.empty((57, h, w), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    be.upsample_device(d_net.data_ptr(), 57, 46, 46, 8, d_up.data_ptr())
    up = d_up.cpu().numpy()
    heat = np.ascontiguousarray(up[:18])
    paf = np.ascontiguousarray(up[19:])
    thr, maxp = float(np.quantile(heat, 0.9)), 32
    d_heat = torch.from_numpy(heat).cuda()
    d_cnt = torch.zeros(18, dtype=torch.int32, device="cuda")
    d_pk = torch.zeros((18, maxp, 5), dtype=torch.float32, device="cuda")
    be.nms_device(d_heat.data_ptr(), 18, h, w, thr, maxp, d_cnt.data_ptr(), d_pk.data_ptr())
    counts, peaks = d_cnt.cpu().numpy(), d_pk.cpu().numpy()
    parts, pafidx, new_rows = coco_limbs()
    d_paf = torch.from_numpy(paf).cuda()
    d_cand = torch.zeros((19, maxp, maxp, 2), dtype=torch.float32, device="cuda")
    paf_thr = float(np.quantile(np.abs(paf), 0.5))  # random weights: a data-driven threshold exercises both branches
    be.paf_candidates_device(d_paf.data_ptr(), h, w, d_cnt.data_ptr(), d_pk.data_ptr(), maxp, parts, pafidx,
                             paf_thr, d_cand.data_ptr())
    cand = d_cand.cpu().numpy()
    ref = O.paf_candidates(paf, counts, peaks, parts, pafidx, paf_thr)
    assert cand.tobytes() == ref.tobytes()
    got_p, got_s = assemble_people(counts, peaks, cand, parts, new_rows)
    ref_p, ref_s = O.assemble_people(counts, peaks, ref, parts, new_rows)
    assert np.array_equal(got_p, ref_p) and got_s.tobytes() == ref_s.tobytes()
    be.close()
