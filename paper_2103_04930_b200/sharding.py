"""Frame-group sharding of a batched FrameData across GPUs.

A FrameData of N frames arrives as channels = 3N (batch folded into channels,
proj/src/server.cpp:297-301). Frames are independent, so a cycle splits into
contiguous frame groups, one per GPU; the pose-net output [N][57][H/8][W/8] is
batch-major, so each group's result is a contiguous slice of the reply and the
"gather" is a host-side placement — no collective. This module is the Python
statement of the partition the C++ B200Backend split policy uses
(csrc/host/b200_backend.cpp), shared by bench.py's multi-rank runs and tested
with a gloo world on CPU (tests/test_sharding.py).
"""
from __future__ import annotations

from typing import List, Tuple


def frame_groups(n_frames: int, world: int) -> List[Tuple[int, int]]:
    """(first_frame, count) per rank: contiguous, sizes differ by at most one,
    earlier ranks take the remainder — the split order of B200Backend."""
    if n_frames < 0 or world < 1:
        raise ValueError("need n_frames >= 0 and world >= 1")
    groups, first = [], 0
    for r in range(world):
        n = n_frames // world + (1 if r < n_frames % world else 0)
        groups.append((first, n))
        first += n
    return groups


def slices(n_frames: int, world: int, in_per_frame: int, out_per_frame: int):
    """Element ranges of each rank's input and output slice."""
    out = []
    for first, n in frame_groups(n_frames, world):
        out.append(((first * in_per_frame, (first + n) * in_per_frame),
                    (first * out_per_frame, (first + n) * out_per_frame)))
    return out
