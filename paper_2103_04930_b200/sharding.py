"""Frame-group sharding of a batched FrameData across GPUs.

A FrameData of N frames arrives as channels = 3N (batch folded into channels,
proj/src/server.cpp:297-301). Frames are independent, so a cycle splits into
contiguous frame groups, one per GPU; the pose-net output [N][C][H/8][W/8] is
batch-major, so each group's result is a contiguous slice of the reply and the
"gather" is a host-side placement, no collective.

The partition is the product's own: avec_frame_groups in libavec_host.so, the
function B200Backend's split policy calls (csrc/host/b200_backend.cpp).
bench.py's ranks take their frame group from it, and tests/test_sharding.py
checks it on a gloo world.
"""
from __future__ import annotations

import ctypes
from typing import List, Tuple

from ._lib import LIB_DIR, load

_HOST = None


def _host() -> ctypes.CDLL:
    global _HOST
    if _HOST is None:
        load()  # libavec_cuda.so first: libavec_host.so links it
        _HOST = ctypes.CDLL(str(LIB_DIR / "libavec_host.so"))
        _HOST.avec_frame_groups.restype = ctypes.c_int
        _HOST.avec_frame_groups.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    return _HOST


def frame_groups(n_frames: int, groups: int) -> List[Tuple[int, int]]:
    """(first_frame, count) per group, as B200Backend splits a cycle."""
    if n_frames < 0 or groups < 1:
        raise ValueError("need n_frames >= 0 and groups >= 1")
    first = (ctypes.c_uint64 * groups)()
    count = (ctypes.c_uint64 * groups)()
    if _host().avec_frame_groups(n_frames, groups, first, count) != 0:
        raise ValueError("avec_frame_groups failed")
    return [(int(first[g]), int(count[g])) for g in range(groups)]
