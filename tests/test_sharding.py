"""N>1 path on CPU: world_size-2 gloo ranks shard a batched cycle into frame
groups with the PRODUCT partition (avec_frame_groups in libavec_host.so, the
function B200Backend's split policy calls), each computes its slice, rank 0
assembles; the result must equal the unsharded computation bit for bit (the
per-frame op here is the oracle's conv layer, standing in for the pose net
whose frames are independent; the GPU split itself is checked in
tests/test_gpu_multi.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_04930_b200.sharding import frame_groups


def test_frame_groups_cover_exactly():
    for n in range(0, 40):
        for w in range(1, 9):
            g = frame_groups(n, w)
            assert len(g) == w and sum(c for _, c in g) == n
            assert all(g[i][0] + g[i][1] == g[i + 1][0] for i in range(w - 1))
            assert max(c for _, c in g) - min(c for _, c in g) <= 1
    assert frame_groups(32, 8) == [(4 * i, 4) for i in range(8)]  # C5: 32 frames on 8 B200
    assert frame_groups(8, 3) == [(0, 3), (3, 3), (6, 2)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _per_frame_op(frames):
    import oracle_lib as O
    rng = np.random.default_rng(5)
    w = rng.standard_normal((8, 3, 3, 3)).astype(np.float32)
    b = rng.standard_normal(8).astype(np.float32)
    x = frames.transpose(0, 2, 3, 1)  # NCHW -> NHWC
    return O.conv2d_nhwc(np.ascontiguousarray(x), w, b, relu=True, round_bf16=True).transpose(0, 3, 1, 2)


def _rank(rank, world, port, n_frames, q):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, W = 16, 24
    rng = np.random.default_rng(11)
    batch = rng.random((n_frames, 3, H, W), dtype=np.float32)
    first, n = frame_groups(n_frames, world)[rank]
    mine = _per_frame_op(batch[first:first + n]) if n else np.zeros((0, 8, H, W), np.float32)
    # uneven groups: pad to the largest, gather, trim (host-side placement only)
    cap = max(c for _, c in frame_groups(n_frames, world))
    buf = np.zeros((cap, 8, H, W), np.float32)
    buf[:n] = mine
    out = [torch.zeros(cap, 8, H, W) for _ in range(world)]
    dist.all_gather(out, torch.from_numpy(buf))
    if rank == 0:
        parts = [out[r][:c].numpy() for r, (_, c) in enumerate(frame_groups(n_frames, world))]
        got = np.concatenate(parts)
        want = _per_frame_op(batch)
        q.put(bool(got.tobytes() == want.tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [8, 5])
def test_gloo_two_ranks_match_unsharded(n_frames):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_frame_groups_are_batch_major_output_slices():
    # C2 batch of 8 on 2 GPUs: each GPU's reply is one contiguous range of the output
    per = 57 * 46 * 82
    g = frame_groups(8, 2)
    assert [(f * per, (f + n) * per) for f, n in g] == [(0, 4 * per), (4 * per, 8 * per)]
