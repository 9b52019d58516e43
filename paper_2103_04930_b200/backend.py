"""Python mirror of the reference plugin interface, backed by the B200 C-ABI.

Reference: accelfwd::backend (proj/include/accelfwd/backend.hpp:20-99) and
accelfwd::wire model types (proj/include/accelfwd/wire.hpp:28-87). Names,
argument meaning and error behaviour follow the reference so tests read like
proj/tests/test_backend.cpp:
  * register_model is idempotent per digest, handles start at 1;
  * forward raises AvecError(name="unknown_model") for foreign handles,
    AvecError(name="degenerate_output") for K<1 or K>E, ValueError (the
    reference's std::invalid_argument) when data size disagrees with dims.
"""
from __future__ import annotations

import ctypes
import dataclasses
import hashlib
import struct
from typing import Optional

import numpy as np

from . import _lib


@dataclasses.dataclass(frozen=True)
class Dims:
    """wire::Dims (wire.hpp:28-42)."""
    batch: int = 1
    channels: int = 1
    height: int = 1
    width: int = 1

    def elem_count(self) -> int:
        return self.batch * self.channels * self.height * self.width

    def valid(self) -> bool:
        return (self.batch >= 1 and self.channels >= 1 and 1 <= self.height <= 65535
                and 1 <= self.width <= 65535)


def model_digest(structure: bytes, weights: bytes, output_divisor: float) -> bytes:
    """sha256(structure || weights || divisor as 8-byte LE double) — wire.cpp:70-79."""
    h = hashlib.sha256()
    h.update(structure)
    h.update(weights)
    h.update(struct.pack("<d", output_divisor))
    return h.digest()


@dataclasses.dataclass
class ModelDescriptor:
    """wire::ModelDescriptor (wire.hpp:73-79)."""
    name: str
    structure: bytes
    weights: bytes
    output_divisor: float
    digest: bytes


def make_model(name: str, structure: bytes, weights: bytes, output_divisor: float) -> ModelDescriptor:
    """wire::make_model (wire.cpp:81-92): rejects divisor <= 0."""
    if not output_divisor > 0.0:
        raise _lib.AvecError(3, "output divisor must be > 0")
    return ModelDescriptor(name, bytes(structure), bytes(weights), float(output_divisor),
                           model_digest(structure, weights, output_divisor))


@dataclasses.dataclass
class Frame:
    """backend::Frame (backend.hpp:22-25): flattened, batch-major fp32."""
    dims: Dims
    data: np.ndarray


@dataclasses.dataclass
class Heatmap:
    """backend::Heatmap (backend.hpp:27-30)."""
    data: np.ndarray

    def elem_count(self) -> int:
        return int(self.data.size)


@dataclasses.dataclass(frozen=True)
class ModelHandle:
    """backend::ModelHandle (backend.hpp:34-37): valid ids start at 1."""
    id: int = 0


def output_elems(input_elems: int, divisor: float) -> int:
    """wire::output_elems (wire.cpp:18-22): round half away from zero."""
    if not divisor > 0.0:
        raise ValueError("output divisor must be > 0")
    k = input_elems / divisor
    return int(np.floor(k + 0.5)) if k >= 0 else -int(np.floor(-k + 0.5))


def device_count() -> int:
    L = _lib.load()
    n = ctypes.c_int(0)
    _lib.check(L.avec_device_count(ctypes.byref(n)))
    return n.value


class B200Backend:
    """Backend implementation on one B200 (one avec_ctx)."""

    def __init__(self, device: int = 0, slots: int = 2):
        self._L = _lib.load()
        ctx = ctypes.c_void_p()
        _lib.check(self._L.avec_ctx_create(device, slots, ctypes.byref(ctx)))
        self._ctx = ctx
        self.device = device

    def close(self) -> None:
        if self._ctx:
            self._L.avec_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ctx(self) -> ctypes.c_void_p:
        return self._ctx

    def label(self) -> str:
        return self._L.avec_ctx_label(self._ctx).decode()

    def register_model(self, model: ModelDescriptor) -> ModelHandle:
        h = ctypes.c_uint64(0)
        u8 = ctypes.POINTER(ctypes.c_uint8)
        dig = (ctypes.c_uint8 * 32).from_buffer_copy(model.digest)
        s = (ctypes.c_uint8 * max(len(model.structure), 1)).from_buffer_copy(model.structure or b"\0")
        w = (ctypes.c_uint8 * max(len(model.weights), 1)).from_buffer_copy(model.weights or b"\0")
        name = model.name.encode()
        _lib.check(self._L.avec_model_register(
            self._ctx, ctypes.cast(dig, u8), name, len(name), ctypes.cast(s, u8), len(model.structure),
            ctypes.cast(w, u8), len(model.weights), model.output_divisor, ctypes.byref(h)))
        return ModelHandle(h.value)

    def model_kind(self, handle: ModelHandle) -> int:
        k = ctypes.c_int(-1)
        _lib.check(self._L.avec_model_kind(self._ctx, handle.id, ctypes.byref(k)))
        return k.value

    def output_elems(self, handle: ModelHandle, dims: Dims) -> int:
        k = ctypes.c_uint64(0)
        _lib.check(self._L.avec_output_elems(self._ctx, handle.id, dims.batch, dims.channels,
                                             dims.height, dims.width, ctypes.byref(k)))
        return k.value

    def forward(self, handle: ModelHandle, frame: Frame, out: Optional[np.ndarray] = None,
                timing: Optional[list] = None) -> Heatmap:
        """Backend::forward on host buffers (H2D, kernels, D2H inside)."""
        data = np.ascontiguousarray(frame.data, dtype=np.float32).ravel()
        d = frame.dims
        if data.size != d.elem_count():
            raise ValueError("frame data size disagrees with dims")
        k = self.output_elems(handle, d)
        if out is None:
            out = np.empty(k, np.float32)
        secs = ctypes.c_double(0)
        _lib.check(self._L.avec_forward(self._ctx, handle.id, d.batch, d.channels, d.height, d.width,
                                        data.ctypes.data, data.size, out.ctypes.data, out.size,
                                        ctypes.byref(secs)))
        if timing is not None:
            timing.append(secs.value)
        return Heatmap(out)

    def forward_device(self, handle: ModelHandle, dims: Dims, d_in: int, d_out: int,
                       stream: int = 0) -> None:
        """Device-resident forward (pointers of this GPU), enqueued on `stream`."""
        _lib.check(self._L.avec_forward_device(self._ctx, handle.id, dims.batch, dims.channels,
                                               dims.height, dims.width, d_in, d_out,
                                               ctypes.c_void_p(stream) if stream else None))

    # ---- pose-net extras ----
    def num_layers(self, handle: ModelHandle) -> int:
        n = ctypes.c_int(0)
        _lib.check(self._L.avec_posenet_num_layers(self._ctx, handle.id, ctypes.byref(n)))
        return n.value

    def layer_info(self, handle: ModelHandle, layer: int) -> dict:
        vals = [ctypes.c_int(0) for _ in range(5)]
        _lib.check(self._L.avec_posenet_layer_info(self._ctx, handle.id, layer,
                                                   *[ctypes.byref(v) for v in vals]))
        return dict(zip(["cin", "cout", "k", "level", "relu"], [v.value for v in vals]))

    def layer_out_level(self, handle: ModelHandle, dims: Dims, layer: int) -> int:
        """Pyramid level of the layer's output as the plan stores it (one more
        than the layer's own level when its 2x2 max-pool is fused)."""
        lv = ctypes.c_int(0)
        _lib.check(self._L.avec_posenet_layer_out_level(self._ctx, handle.id, dims.batch, dims.channels,
                                                        dims.height, dims.width, layer, ctypes.byref(lv)))
        return lv.value

    def layer_fusion(self, handle: ModelHandle, dims: Dims, layer: int):
        """(kind, in_layer): 0 plain, 1 pooled output, 2 fused into the next
        layer (no output of its own), 3 second layer of a fused head whose
        input is layer `in_layer`'s input (avec_posenet_layer_fusion)."""
        kind, src = ctypes.c_int(0), ctypes.c_int(0)
        _lib.check(self._L.avec_posenet_layer_fusion(self._ctx, handle.id, dims.batch, dims.channels, dims.height,
                                                     dims.width, layer, ctypes.byref(kind), ctypes.byref(src)))
        return kind.value, src.value

    def layer_io(self, handle: ModelHandle, frame: Frame, layer: int):
        """(input, output) activations of conv `layer`, unpadded fp32 NHWC; the
        output is the pooled tensor for layers with a fused max-pool."""
        info = self.layer_info(handle, layer)
        d = frame.dims
        n_img = d.batch * d.channels // 3
        hl, wl = d.height >> info["level"], d.width >> info["level"]
        ol = self.layer_out_level(handle, d, layer)
        _, src = self.layer_fusion(handle, d, layer)
        cin = self.layer_info(handle, src)["cin"]
        lin = np.empty((n_img, hl, wl, cin), np.float32)
        lout = np.empty((n_img, d.height >> ol, d.width >> ol, info["cout"]), np.float32)
        data = np.ascontiguousarray(frame.data, np.float32).ravel()
        _lib.check(self._L.avec_posenet_layer_io(self._ctx, handle.id, d.batch, d.channels, d.height,
                                                 d.width, data.ctypes.data, layer, lin.ctypes.data,
                                                 lin.size, lout.ctypes.data, lout.size))
        return lin, lout

    def layer_rows(self, handle: ModelHandle, frame: Frame, layer: int, in_rows, out_rows):
        """Selected rows of conv `layer`'s input and output views
        (avec_posenet_layer_rows): `in_rows` / `out_rows` are (image, y) pairs;
        rows outside the image come back as zeros. Returns fp32 arrays
        [len(in_rows)][W_in][cin] and [len(out_rows)][W_out][cout]."""
        info = self.layer_info(handle, layer)
        d = frame.dims
        ol = self.layer_out_level(handle, d, layer)
        _, src = self.layer_fusion(handle, d, layer)
        cin = self.layer_info(handle, src)["cin"]
        ir = np.ascontiguousarray(np.asarray(in_rows, np.int32).reshape(-1, 2))
        orr = np.ascontiguousarray(np.asarray(out_rows, np.int32).reshape(-1, 2))
        lin = np.empty((len(ir), d.width >> info["level"], cin), np.float32)
        lout = np.empty((len(orr), d.width >> ol, info["cout"]), np.float32)
        data = np.ascontiguousarray(frame.data, np.float32).ravel()
        _lib.check(self._L.avec_posenet_layer_rows(self._ctx, handle.id, d.batch, d.channels, d.height, d.width,
                                                   data.ctypes.data, layer, len(ir), ir.ctypes.data,
                                                   lin.ctypes.data, len(orr), orr.ctypes.data, lout.ctypes.data))
        return lin, lout

    def profile(self, handle: ModelHandle, dims: Dims, d_in: int, reps: int = 3) -> list:
        """Per-launch device timings of the pose-net plan (see avec_posenet_profile)."""
        n = ctypes.c_int(0)
        cap = 256
        kind = np.zeros(cap, np.int32)
        flops = np.zeros(cap, np.float64)
        nbytes = np.zeros(cap, np.float64)
        ms = np.zeros(cap, np.float32)
        _lib.check(self._L.avec_posenet_profile(
            self._ctx, handle.id, dims.batch, dims.channels, dims.height, dims.width, d_in, reps, cap,
            ctypes.byref(n), kind.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), flops.ctypes.data,
            nbytes.ctypes.data, ms.ctypes.data))
        names = {0: "conv_first", 1: "conv_pm", 2: "maxpool", 3: "conv_tc", 4: "conv_head", 5: "conv12"}
        return [dict(kind=names[int(kind[i])], flops=float(flops[i]), bytes=float(nbytes[i]),
                     ms=float(ms[i])) for i in range(n.value)]

    def upsample_device(self, d_in: int, planes: int, h: int, w: int, scale: int, d_out: int,
                        stream: int = 0) -> None:
        _lib.check(self._L.avec_upsample_device(self._ctx, d_in, planes, h, w, scale, d_out,
                                                ctypes.c_void_p(stream) if stream else None))

    def paf_candidates_device(self, d_paf: int, h: int, w: int, d_counts: int, d_peaks: int, max_peaks: int,
                              limb_parts: np.ndarray, limb_paf: np.ndarray, threshold: float, d_cand: int,
                              stream: int = 0) -> None:
        """Score every candidate limb on the device (avec_paf_candidates_device)."""
        lp = np.ascontiguousarray(limb_parts, np.int32)
        lf = np.ascontiguousarray(limb_paf, np.int32)
        _lib.check(self._L.avec_paf_candidates_device(self._ctx, d_paf, h, w, d_counts, d_peaks, max_peaks,
                                                      lp.ctypes.data, lf.ctypes.data, lp.shape[0], threshold, d_cand,
                                                      ctypes.c_void_p(stream) if stream else None))

    def upsample_nms_device(self, d_in: int, planes: int, h: int, w: int, scale: int, threshold: float,
                            max_peaks: int, d_out: int, d_counts: int, d_peaks: int, stream: int = 0) -> None:
        """upsample_device + nms_device of its output in one pass (avec_upsample_nms_device)."""
        _lib.check(self._L.avec_upsample_nms_device(self._ctx, d_in, planes, h, w, scale, threshold, max_peaks,
                                                    d_out, d_counts, d_peaks,
                                                    ctypes.c_void_p(stream) if stream else None))

    def nms_device(self, d_in: int, planes: int, h: int, w: int, threshold: float, max_peaks: int,
                   d_counts: int, d_peaks: int, stream: int = 0) -> None:
        _lib.check(self._L.avec_nms_device(self._ctx, d_in, planes, h, w, threshold, max_peaks,
                                           d_counts, d_peaks,
                                           ctypes.c_void_p(stream) if stream else None))


class PipelineStream:
    """Pipelined cycle on one GPU (avec_stream_*): frames land front to back
    in a pinned buffer, feed() reports landed bytes, finish() returns the
    device compute seconds once the pinned output is complete."""

    def __init__(self, backend: B200Backend):
        self._L = backend._L
        self._be = backend  # keeps the context alive
        s = ctypes.c_void_p()
        _lib.check(self._L.avec_stream_create(backend.ctx, ctypes.byref(s)))
        self._s = s

    def begin(self, handle: ModelHandle, dims: Dims, in_ptr: int, out_ptr: int, out_elems: int) -> None:
        _lib.check(self._L.avec_stream_begin(self._s, handle.id, dims.batch, dims.channels, dims.height, dims.width,
                                             in_ptr, out_ptr, out_elems))

    def feed(self, landed_bytes: int) -> None:
        _lib.check(self._L.avec_stream_feed(self._s, landed_bytes))

    def finish(self) -> float:
        secs = ctypes.c_double(0)
        _lib.check(self._L.avec_stream_finish(self._s, ctypes.byref(secs)))
        return secs.value

    def abort(self) -> None:
        _lib.check(self._L.avec_stream_abort(self._s))

    def close(self) -> None:
        if self._s:
            self._L.avec_stream_destroy(self._s)
            self._s = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def coco_limbs():
    """OpenPose COCO limb types: (limb_parts [19,2], limb_paf [19,2], new_row_limbs)."""
    L = _lib.load()
    parts = np.zeros((19, 2), np.int32)
    paf = np.zeros((19, 2), np.int32)
    n, new_rows = ctypes.c_int(0), ctypes.c_int(0)
    _lib.check(L.avec_coco_limbs(parts.ctypes.data, paf.ctypes.data, ctypes.byref(n), ctypes.byref(new_rows)))
    return parts, paf, new_rows.value


def assemble_people(counts: np.ndarray, peaks: np.ndarray, cand: np.ndarray, limb_parts: np.ndarray,
                    new_row_limbs: int, max_people: int = 64):
    """Host person assembly (avec_assemble_people) -> (people [n][parts], scores [n][2])."""
    L = _lib.load()
    counts = np.ascontiguousarray(counts, np.int32)
    peaks = np.ascontiguousarray(peaks, np.float32)
    cand = np.ascontiguousarray(cand, np.float32)
    limb_parts = np.ascontiguousarray(limb_parts, np.int32)
    n_parts, max_peaks = peaks.shape[0], peaks.shape[1]
    people = np.full((max_people, n_parts), -1, np.int32)
    score = np.zeros((max_people, 2), np.float32)
    n = ctypes.c_int(0)
    _lib.check(L.avec_assemble_people(counts.ctypes.data, peaks.ctypes.data, n_parts, max_peaks, cand.ctypes.data,
                                      limb_parts.ctypes.data, limb_parts.shape[0], new_row_limbs, max_people,
                                      people.ctypes.data, score.ctypes.data, ctypes.byref(n)))
    return people[:n.value], score[:n.value]


def synth_posenet_weights(structure: bytes) -> np.ndarray:
    """The engine's deterministic init for a spec (Caffe-order fp32 blob)."""
    L = _lib.load()
    n = ctypes.c_uint64(0)
    u8 = ctypes.POINTER(ctypes.c_uint8)
    s = (ctypes.c_uint8 * len(structure)).from_buffer_copy(structure)
    _lib.check(L.avec_posenet_synth_weights(ctypes.cast(s, u8), len(structure), None, ctypes.byref(n)))
    out = np.empty(n.value, np.float32)
    _lib.check(L.avec_posenet_synth_weights(ctypes.cast(s, u8), len(structure),
                                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                            ctypes.byref(n)))
    return out


class PinnedBuffer:
    """Page-locked host buffer from avec_host_alloc, viewed as a numpy array."""

    def __init__(self, n: int, dtype=np.float32):
        self._L = _lib.load()
        nbytes = int(n) * np.dtype(dtype).itemsize
        self.ptr = self._L.avec_host_alloc(max(nbytes, 1))
        if not self.ptr:
            raise MemoryError(self._L.avec_last_error().decode())
        buf = (ctypes.c_uint8 * max(nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(n))

    def free(self):
        if self.ptr:
            self.array = None
            self._L.avec_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
