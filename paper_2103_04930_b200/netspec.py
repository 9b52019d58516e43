"""Pose-net spec strings and layer tables (mirror of csrc/cuda/netspec.cpp).

openpose_coco: OpenPose pose_deploy_linevec.prototxt — VGG-19's first ten
convolutions, conv4_3_CPM/conv4_4_CPM, a stage-1 two-branch block (3x3 convs)
and stages 2..6 (7x7 convs) fed by concat(L1, L2, trunk); L1 = 38 PAF
channels, L2 = 19 heatmap channels. Wire output [19 heat | 38 PAF].

openpose_body25: OpenPose body_25/pose_deploy.prototxt (restated from the
public prototxt's structure): PReLU from conv4_2 on; 4 PAF stages (L2) then 2
heatmap stages (L1), each five dense blocks of three 3x3 convs concatenated
(width 96 in the first stage of each branch, 128 after) + Mconv6/Mconv7 1x1.
52 PAF + 26 heatmap channels; wire output [26 heat | 52 PAF].

Weights blob (Caffe order, fp32): per conv W[cout][cin][k][k], bias[cout], and
for PReLU layers slope[cout].
"""
from __future__ import annotations

import dataclasses
from typing import List

import numpy as np

PAF, HEAT, TRUNK = 38, 19, 128
OUT_CHANNELS = PAF + HEAT
COCO_DIVISOR = 192.0 / 57.0  # = 3*8*8/57: K = round(E/c) is exactly the net's output size
B25_PAF, B25_HEAT = 52, 26
BODY25_DIVISOR = 192.0 / 78.0
ACT_NONE, ACT_RELU, ACT_PRELU = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class ConvDef:
    name: str
    cin: int
    cout: int
    k: int
    act: int
    level: int

    @property
    def relu(self) -> int:  # backwards-compatible alias of `act`
        return self.act


def spec(family: str = "openpose_coco", stages: int = 6, seed: int = 1, input_dtype: str = "bf16") -> bytes:
    """avecnet structure bytes. input_dtype "tf32": conv1_1 consumes the fp32
    frames as tf32 tensor-core operands instead of bf16 (conv_first.cu)."""
    lines = ["avecnet 1", f"family {family}"]
    if stages != 6:
        lines.append(f"stages {stages}")
    if input_dtype != "bf16":
        if input_dtype != "tf32":
            raise ValueError("input_dtype must be bf16 or tf32")
        lines.append("input tf32")
    lines.append(f"init he_uniform {seed}")
    return ("\n".join(lines) + "\n").encode()


def _trunk(late_act: int) -> List[ConvDef]:
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
    add("conv4_2", 512, 512, 3, late_act, 3)
    add("conv4_3_CPM", 512, 256, 3, late_act, 3)
    add("conv4_4_CPM", 256, 128, 3, late_act, 3)
    return L


def coco_layers(stages: int = 6) -> List[ConvDef]:
    L = _trunk(ACT_RELU)
    add = lambda *a: L.append(ConvDef(*a))
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


def body25_layers() -> List[ConvDef]:
    L = _trunk(ACT_PRELU)

    def stage(sfx, cin, w, c6, out):
        for blk in range(1, 6):
            for j in range(3):
                ci = w if j else (cin if blk == 1 else 3 * w)
                L.append(ConvDef(f"Mconv{blk}{sfx}_{j}", ci, w, 3, ACT_PRELU, 3))
        L.append(ConvDef("Mconv6" + sfx, 3 * w, c6, 1, ACT_PRELU, 3))
        L.append(ConvDef("Mconv7" + sfx, c6, out, 1, ACT_NONE, 3))

    stage("_stage0_L2", TRUNK, 96, 256, B25_PAF)
    for t in (1, 2, 3):
        stage(f"_stage{t}_L2", TRUNK + B25_PAF, 128, 512, B25_PAF)
    stage("_stage0_L1", TRUNK + B25_PAF, 96, 256, B25_HEAT)
    stage("_stage1_L1", TRUNK + B25_HEAT + B25_PAF, 128, 512, B25_HEAT)
    return L


def layers_for(family: str) -> List[ConvDef]:
    return body25_layers() if family == "openpose_body25" else coco_layers()


def weight_floats(layers: List[ConvDef]) -> int:
    return sum(c.cout * c.cin * c.k * c.k + c.cout + (c.cout if c.act == ACT_PRELU else 0) for c in layers)


def split_weights(layers: List[ConvDef], blob: np.ndarray):
    """Caffe-order blob -> [(W[cout][cin][k][k], b[cout], slope[cout] or None)] per layer."""
    out, off = [], 0
    for c in layers:
        n = c.cout * c.cin * c.k * c.k
        w = blob[off:off + n].reshape(c.cout, c.cin, c.k, c.k)
        off += n
        b = blob[off:off + c.cout]
        off += c.cout
        s = None
        if c.act == ACT_PRELU:
            s = blob[off:off + c.cout]
            off += c.cout
        out.append((w, b, s))
    assert off == blob.size
    return out


def macs_per_pixel(layers: List[ConvDef]) -> float:
    """Multiply-accumulates per INPUT pixel (1,003,766 COCO, 594,970 BODY_25)."""
    return sum(c.cin * c.cout * c.k * c.k / (4 ** c.level) for c in layers)


def flops_per_frame(layers: List[ConvDef], h: int, w: int) -> float:
    return 2.0 * sum(c.cin * c.cout * c.k * c.k * (h >> c.level) * (w >> c.level) for c in layers)
