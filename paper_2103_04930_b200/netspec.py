"""Pose-net spec strings and the COCO layer table (mirror of csrc/cuda/netspec.cpp).

The table follows OpenPose's pose_deploy_linevec.prototxt (COCO): VGG-19's
first ten convolutions, conv4_3_CPM/conv4_4_CPM, a stage-1 two-branch block
(3x3 convs) and stages 2..6 (7x7 convs) fed by concat(L1, L2, trunk).
L1 = 38 PAF channels, L2 = 19 heatmap channels. The weights blob is Caffe-order
fp32: per conv W[cout][cin][kh][kw] then bias[cout].
"""
from __future__ import annotations

import dataclasses
from typing import List

import numpy as np

PAF, HEAT, TRUNK = 38, 19, 128
OUT_CHANNELS = PAF + HEAT
COCO_DIVISOR = 192.0 / 57.0  # = 3*8*8/57: K = round(E/c) is exactly the net's output size


@dataclasses.dataclass(frozen=True)
class ConvDef:
    name: str
    cin: int
    cout: int
    k: int
    relu: int
    level: int


def spec(family: str = "openpose_coco", stages: int = 6, seed: int = 1) -> bytes:
    lines = ["avecnet 1", f"family {family}"]
    if stages != 6:
        lines.append(f"stages {stages}")
    lines.append(f"init he_uniform {seed}")
    return ("\n".join(lines) + "\n").encode()


def coco_layers(stages: int = 6) -> List[ConvDef]:
    L = []
    add = lambda *a: L.append(ConvDef(*a))
    add("conv1_1", 3, 64, 3, 1, 0)
    add("conv1_2", 64, 64, 3, 1, 0)
    add("conv2_1", 64, 128, 3, 1, 1)
    add("conv2_2", 128, 128, 3, 1, 1)
    add("conv3_1", 128, 256, 3, 1, 2)
    for i in (2, 3, 4):
        add(f"conv3_{i}", 256, 256, 3, 1, 2)
    add("conv4_1", 256, 512, 3, 1, 3)
    add("conv4_2", 512, 512, 3, 1, 3)
    add("conv4_3_CPM", 512, 256, 3, 1, 3)
    add("conv4_4_CPM", 256, 128, 3, 1, 3)
    for b, out in (("_L1", PAF), ("_L2", HEAT)):
        add("conv5_1_CPM" + b, 128, 128, 3, 1, 3)
        add("conv5_2_CPM" + b, 128, 128, 3, 1, 3)
        add("conv5_3_CPM" + b, 128, 128, 3, 1, 3)
        add("conv5_4_CPM" + b, 128, 512, 1, 1, 3)
        add("conv5_5_CPM" + b, 512, out, 1, 0, 3)
    for t in range(2, stages + 1):
        for b, out in (("_L1", PAF), ("_L2", HEAT)):
            sfx = f"_stage{t}{b}"
            add("Mconv1" + sfx, PAF + HEAT + TRUNK, 128, 7, 1, 3)
            for i in range(2, 6):
                add(f"Mconv{i}" + sfx, 128, 128, 7, 1, 3)
            add("Mconv6" + sfx, 128, 128, 1, 1, 3)
            add("Mconv7" + sfx, 128, out, 1, 0, 3)
    return L


def weight_floats(layers: List[ConvDef]) -> int:
    return sum(c.cout * c.cin * c.k * c.k + c.cout for c in layers)


def split_weights(layers: List[ConvDef], blob: np.ndarray):
    """Caffe-order blob -> [(W[cout][cin][k][k], b[cout])] per layer."""
    out, off = [], 0
    for c in layers:
        n = c.cout * c.cin * c.k * c.k
        w = blob[off:off + n].reshape(c.cout, c.cin, c.k, c.k)
        off += n
        b = blob[off:off + c.cout]
        off += c.cout
        out.append((w, b))
    assert off == blob.size
    return out


def macs_per_pixel(layers: List[ConvDef]) -> float:
    """Multiply-accumulates per INPUT pixel (1,003,766 for COCO)."""
    return sum(c.cin * c.cout * c.k * c.k / (4 ** c.level) for c in layers)


def flops_per_frame(layers: List[ConvDef], h: int, w: int) -> float:
    return 2.0 * sum(c.cin * c.cout * c.k * c.k * (h >> c.level) * (w >> c.level) for c in layers)
