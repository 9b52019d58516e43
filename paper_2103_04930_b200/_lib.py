"""Loader for the in-tree C-ABI library (include/avec_cuda.h).

There is no fallback: if libavec_cuda.so is missing or cannot load, every
entry point raises. The product path never touches the oracle.
"""
from __future__ import annotations

import ctypes
import pathlib

PKG = pathlib.Path(__file__).resolve().parent
LIB_DIR = PKG / "lib"

AVEC_OK = 0
ERROR_NAMES = {
    1: "invalid_argument",
    2: "unknown_model",
    3: "invalid_model",
    4: "degenerate_output",
    5: "cuda",
    6: "out_of_memory",
    7: "unsupported",
}

AVEC_MODEL_MOCKPOSE = 0
AVEC_MODEL_POSENET = 1

# every symbol include/avec_cuda.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "avec_last_error", "avec_version", "avec_device_count", "avec_ctx_create",
    "avec_ctx_destroy", "avec_ctx_label", "avec_model_register", "avec_model_kind",
    "avec_output_elems", "avec_forward", "avec_forward_device", "avec_upsample_device",
    "avec_nms_device", "avec_upsample_nms_device", "avec_posenet_layer_io", "avec_posenet_layer_rows", "avec_posenet_layer_out_level", "avec_posenet_layer_fusion", "avec_posenet_layer_info",
    "avec_posenet_num_layers", "avec_posenet_profile", "avec_posenet_synth_weights", "avec_host_alloc", "avec_host_free",
    "avec_paf_candidates_device", "avec_assemble_people", "avec_coco_limbs",
    "avec_stream_create", "avec_stream_destroy", "avec_stream_prepare", "avec_stream_begin", "avec_stream_feed", "avec_stream_finish",
    "avec_stream_abort",
]

_lib = None


class AvecLibraryMissing(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = LIB_DIR / "libavec_cuda.so"
    if not path.exists():
        raise AvecLibraryMissing(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` or `make product`")
    L = ctypes.CDLL(str(path))
    c = ctypes
    vp, u8p, u64, u32, i, d = c.c_void_p, c.POINTER(c.c_uint8), c.c_uint64, c.c_uint32, c.c_int, c.c_double
    fp = c.POINTER(c.c_float)
    sig = {
        "avec_last_error": (c.c_char_p, []),
        "avec_version": (c.c_char_p, []),
        "avec_device_count": (i, [c.POINTER(i)]),
        "avec_ctx_create": (i, [i, i, c.POINTER(vp)]),
        "avec_ctx_destroy": (None, [vp]),
        "avec_ctx_label": (c.c_char_p, [vp]),
        "avec_model_register": (i, [vp, u8p, c.c_char_p, c.c_size_t, u8p, c.c_size_t, u8p, u64, d,
                                    c.POINTER(u64)]),
        "avec_model_kind": (i, [vp, u64, c.POINTER(i)]),
        "avec_output_elems": (i, [vp, u64, u32, u32, u32, u32, c.POINTER(u64)]),
        "avec_forward": (i, [vp, u64, u32, u32, u32, u32, vp, u64, vp, u64, c.POINTER(d)]),
        "avec_forward_device": (i, [vp, u64, u32, u32, u32, u32, vp, vp, vp]),
        "avec_upsample_device": (i, [vp, vp, i, i, i, i, vp, vp]),
        "avec_nms_device": (i, [vp, vp, i, i, i, c.c_float, i, vp, vp, vp]),
        "avec_upsample_nms_device": (i, [vp, vp, i, i, i, i, c.c_float, i, vp, vp, vp, vp]),
        "avec_posenet_layer_io": (i, [vp, u64, u32, u32, u32, u32, vp, i, vp, u64, vp, u64]),
        "avec_posenet_layer_rows": (i, [vp, u64, u32, u32, u32, u32, vp, i, i, vp, vp, i, vp, vp]),
        "avec_posenet_layer_out_level": (i, [vp, u64, u32, u32, u32, u32, i, c.POINTER(i)]),
        "avec_posenet_layer_fusion": (i, [vp, u64, u32, u32, u32, u32, i, c.POINTER(i), c.POINTER(i)]),
        "avec_paf_candidates_device": (i, [vp, vp, i, i, vp, vp, i, vp, vp, i, c.c_float, vp, vp]),
        "avec_assemble_people": (i, [vp, vp, i, i, vp, vp, i, i, i, vp, vp, c.POINTER(i)]),
        "avec_coco_limbs": (i, [vp, vp, c.POINTER(i), c.POINTER(i)]),
        "avec_posenet_layer_info": (i, [vp, u64, i] + [c.POINTER(i)] * 5),
        "avec_posenet_num_layers": (i, [vp, u64, c.POINTER(i)]),
        "avec_posenet_profile": (i, [vp, u64, u32, u32, u32, u32, vp, i, i, c.POINTER(i), vp, vp, vp, vp]),
        "avec_posenet_synth_weights": (i, [u8p, c.c_size_t, fp, c.POINTER(u64)]),
        "avec_host_alloc": (vp, [u64]),
        "avec_stream_create": (i, [vp, c.POINTER(vp)]),
        "avec_stream_destroy": (None, [vp]),
        "avec_stream_prepare": (i, [vp, u64, u32, u32, u32, u32]),
        "avec_stream_begin": (i, [vp, u64, u32, u32, u32, u32, vp, vp, u64]),
        "avec_stream_feed": (i, [vp, u64]),
        "avec_stream_finish": (i, [vp, c.POINTER(d)]),
        "avec_stream_abort": (i, [vp]),
        "avec_host_free": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class AvecError(Exception):
    """Error raised by the engine; `.name` mirrors accelfwd::ErrorCode where one exists."""

    def __init__(self, code: int, message: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {message}")
        self.code = code
        self.name = ERROR_NAMES.get(code, str(code))
        self.message = message


def check(rc: int) -> None:
    if rc != AVEC_OK:
        msg = load().avec_last_error().decode(errors="replace")
        if rc == 1:  # std::invalid_argument in the reference (backend.cpp:92-93)
            raise ValueError(msg)
        raise AvecError(rc, msg)
