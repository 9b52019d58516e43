"""ctypes view of oracle/liboracle.so — the CPU checker (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module. The product (paper_2103_04930_b200) never does.
"""
import ctypes
import pathlib

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
_LIB = None

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def lib():
    global _LIB
    if _LIB is None:
        path = ROOT / "oracle" / "liboracle.so"
        if not path.exists():
            raise RuntimeError(f"{path} missing: run `make -C oracle oracle`")
        L = ctypes.CDLL(str(path))
        u64, u32, i, d = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
        L.oracle_output_elems.argtypes = [u64, d]
        L.oracle_output_elems.restype = u64
        L.oracle_transfer_size.argtypes = [u32, u32, u32, u32, d]
        L.oracle_transfer_size.restype = u64
        L.oracle_segment_means.argtypes = [f32p, u64, d, f64p, u64]
        L.oracle_segment_means.restype = i
        L.oracle_mockpose_forward.argtypes = [f32p, u64, d, f32p, u64]
        L.oracle_mockpose_forward.restype = i
        L.oracle_gen_frame.argtypes = [u64, u32, u32, u32, f32p]
        L.oracle_synth_blobs.argtypes = [u64, u8p, ctypes.c_size_t, u8p, ctypes.c_size_t]
        L.oracle_bf16_round.argtypes = [ctypes.c_float]
        L.oracle_bf16_round.restype = ctypes.c_float
        L.oracle_conv2d_nhwc.argtypes = [f32p, i, i, i, i, f32p, f32p, i, i, i, f32p, i, f32p]
        L.oracle_conv2d_rows.argtypes = [f32p, i, i, i, i, f32p, f32p, i, i, f32p, i, f32p]
        L.oracle_maxpool2_nhwc.argtypes = [f32p, i, i, i, i, f32p]
        L.oracle_upsample_plane.argtypes = [f32p, i, i, i, f32p]
        L.oracle_nms_plane.argtypes = [f32p, i, i, ctypes.c_float, i, i32p, f32p, f32p]
        L.oracle_nms_plane.restype = i
        L.oracle_paf_candidates.argtypes = [f32p, i, i, i32p, f32p, i, i32p, i32p, i, ctypes.c_float, f32p]
        L.oracle_assemble_people.argtypes = [i32p, f32p, i, i, f32p, i32p, i, i, i, i32p, f32p]
        L.oracle_assemble_people.restype = i
        _LIB = L
    return _LIB


def output_elems(e: int, c: float) -> int:
    return int(lib().oracle_output_elems(e, c))


def transfer_size(n, c, h, w, divisor) -> int:
    return int(lib().oracle_transfer_size(n, c, h, w, divisor))


class OracleError(Exception):
    pass


def segment_means(data: np.ndarray, divisor: float) -> np.ndarray:
    data = np.ascontiguousarray(data, np.float32)
    k = output_elems(data.size, divisor)
    out = np.zeros(max(k, 1), np.float64)
    rc = lib().oracle_segment_means(data, data.size, divisor, out, k)
    if rc:
        raise OracleError({1: "empty", 2: "degenerate_output", 3: "size"}[rc])
    return out[:k]


def mockpose_forward(data: np.ndarray, divisor: float) -> np.ndarray:
    data = np.ascontiguousarray(data, np.float32).ravel()
    k = output_elems(data.size, divisor)
    out = np.zeros(max(k, 1), np.float32)
    rc = lib().oracle_mockpose_forward(data, data.size, divisor, out, k)
    if rc:
        raise OracleError({1: "empty", 2: "degenerate_output", 3: "size"}[rc])
    return out[:k]


def gen_frame(seed: int, index: int, width: int, height: int) -> np.ndarray:
    out = np.empty(3 * width * height, np.float32)
    lib().oracle_gen_frame(seed, index, width, height, out)
    return out


def batched_frame(width: int, height: int, batch: int, seed: int = 7, first: int = 0) -> np.ndarray:
    """`batch` harness frames folded into channels (3*batch) — the wire's batching."""
    return np.concatenate([gen_frame(seed, first + b, width, height) for b in range(batch)])


def synth_blobs(seed: int, structure_bytes: int, weights_bytes: int):
    s = np.empty(structure_bytes, np.uint8)
    w = np.empty(weights_bytes, np.uint8)
    lib().oracle_synth_blobs(seed, s, s.size, w, w.size)
    return s.tobytes(), w.tobytes()


def tf32_round(a: np.ndarray) -> np.ndarray:
    """fp32 -> tf32 (10-bit mantissa), round to nearest, ties away from zero:
    cvt.rna.tf32.f32, which conv_first.cu applies to the frames of an
    "input tf32" net (and the upload to its first-layer weights)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    fin = (u & 0x7F800000) != 0x7F800000
    r = np.where(fin, (u + 0x1000) & 0xFFFFE000, u).astype(np.uint32)
    return r.view(np.float32).reshape(np.shape(a))


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Vectorised RNE fp32 -> bf16 -> fp32 (same rule as oracle_bf16_round)."""
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).reshape(a.shape)


def conv2d_nhwc(x: np.ndarray, w: np.ndarray, b: np.ndarray, relu, round_bf16: bool,
                slope: np.ndarray = None) -> np.ndarray:
    """`relu`: activation code 0 none / 1 ReLU / 2 PReLU (bool True = ReLU);
    PReLU takes the per-channel `slope`."""
    n, h, wd, cin = x.shape
    cout, cin2, k, _ = w.shape
    assert cin == cin2
    act = int(relu)
    if act == 2 and slope is None:
        raise ValueError("PReLU needs slopes")
    sl = np.ascontiguousarray(slope if slope is not None else np.zeros(cout), np.float32)
    out = np.empty((n, h, wd, cout), np.float32)
    lib().oracle_conv2d_nhwc(np.ascontiguousarray(x, np.float32), n, h, wd, cin,
                             np.ascontiguousarray(w, np.float32), np.ascontiguousarray(b, np.float32),
                             cout, k, act, sl, int(round_bf16), out)
    return out


def conv2d_rows(win: np.ndarray, w: np.ndarray, b: np.ndarray, relu, round_bf16: bool,
                slope: np.ndarray = None) -> np.ndarray:
    """Selected output rows: win [rows][k][W][cin] (each row's k-row input
    window, zeros outside the image) -> [rows][W][cout]; same arithmetic as
    conv2d_nhwc (oracle_conv2d_rows)."""
    r, k, wd, cin = win.shape
    cout, cin2, k2, _ = w.shape
    assert cin == cin2 and k == k2
    act = int(relu)
    sl = np.ascontiguousarray(slope if slope is not None else np.zeros(cout), np.float32)
    out = np.empty((r, wd, cout), np.float32)
    if r:
        lib().oracle_conv2d_rows(np.ascontiguousarray(win, np.float32), r, k, wd, cin,
                                 np.ascontiguousarray(w, np.float32), np.ascontiguousarray(b, np.float32),
                                 cout, act, sl, int(round_bf16), out)
    return out


def maxpool2_nhwc(x: np.ndarray) -> np.ndarray:
    n, h, w, c = x.shape
    out = np.empty((n, h // 2, w // 2, c), np.float32)
    lib().oracle_maxpool2_nhwc(np.ascontiguousarray(x, np.float32), n, h, w, c, out)
    return out


def upsample_plane(x: np.ndarray, scale: int) -> np.ndarray:
    h, w = x.shape
    out = np.empty((h * scale, w * scale), np.float32)
    lib().oracle_upsample_plane(np.ascontiguousarray(x, np.float32), h, w, scale, out)
    return out


def nms_plane(x: np.ndarray, threshold: float, max_peaks: int):
    h, w = x.shape
    xy = np.zeros(2 * max_peaks, np.int32)
    ref = np.zeros(2 * max_peaks, np.float32)
    sc = np.zeros(max_peaks, np.float32)
    n = lib().oracle_nms_plane(np.ascontiguousarray(x, np.float32), h, w, threshold, max_peaks, xy, ref, sc)
    return xy[: 2 * n].reshape(n, 2), ref[: 2 * n].reshape(n, 2), sc[:n]


def coco_chain(frames_nchw: np.ndarray, layers, wb) -> np.ndarray:
    """Whole COCO pose net on the oracle (bf16 rounding after every layer, as
    the device stores activations), from NCHW fp32 frames [N,3,H,W] to the
    wire output [N][19 heat | 38 PAF][H/8][W/8] flattened."""
    x = bf16_round(frames_nchw.transpose(0, 2, 3, 1) - 0.5)

    def conv(t, idx, final=False):
        w, b, _ = wb[idx]
        return conv2d_nhwc(t, w, b, relu=layers[idx].act, round_bf16=not final)

    cur = conv(x, 0)
    cur = maxpool2_nhwc(conv(cur, 1))
    cur = conv(cur, 2)
    cur = maxpool2_nhwc(conv(cur, 3))
    for j in (4, 5, 6, 7):
        cur = conv(cur, j)
    cur = maxpool2_nhwc(cur)
    for j in (8, 9, 10, 11):
        cur = conv(cur, j)
    trunk = l1 = l2 = cur
    for j in range(12, 17):
        l1 = conv(l1, j)
    for j in range(17, 22):
        l2 = conv(l2, j)
    idx = 22
    for t in range(2, 7):
        cat = np.concatenate([l1, l2, trunk], axis=3)
        a, b_ = cat, cat
        for j in range(7):
            a = conv(a, idx + j, final=(t == 6 and j == 6))
        for j in range(7):
            b_ = conv(b_, idx + 7 + j, final=(t == 6 and j == 6))
        l1, l2 = a, b_
        idx += 14
    return np.concatenate([l2, l1], axis=3).transpose(0, 3, 1, 2).ravel()


def paf_candidates(paf, counts, peaks, limb_parts, limb_paf, thr):
    """Oracle candidate scores [n_limbs][max_peaks][max_peaks][2] (oracle/paf_oracle.c)."""
    paf = np.ascontiguousarray(paf, np.float32)
    counts = np.ascontiguousarray(counts, np.int32)
    peaks = np.ascontiguousarray(peaks, np.float32)
    lp = np.ascontiguousarray(limb_parts, np.int32)
    lf = np.ascontiguousarray(limb_paf, np.int32)
    max_peaks = peaks.shape[1]
    cand = np.zeros((lp.shape[0], max_peaks, max_peaks, 2), np.float32)
    lib().oracle_paf_candidates(paf, paf.shape[1], paf.shape[2], counts, peaks, max_peaks, lp, lf, lp.shape[0],
                                thr, cand)
    return cand


def assemble_people(counts, peaks, cand, limb_parts, new_row_limbs, max_people=64):
    counts = np.ascontiguousarray(counts, np.int32)
    peaks = np.ascontiguousarray(peaks, np.float32)
    cand = np.ascontiguousarray(cand, np.float32)
    lp = np.ascontiguousarray(limb_parts, np.int32)
    people = np.full((max_people, peaks.shape[0]), -1, np.int32)
    score = np.zeros((max_people, 2), np.float32)
    n = lib().oracle_assemble_people(counts, peaks, peaks.shape[0], peaks.shape[1], cand, lp, lp.shape[0],
                                     new_row_limbs, max_people, people, score)
    return people[:n], score[:n]
