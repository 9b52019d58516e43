"""Row-sampled layer parity at full configuration sizes (TEST INFRASTRUCTURE).

At C2 (8x656x368) and C5 (32x1312x736) a whole activation tensor is too big
to compare on the host, and the oracle would take hours on it. Each layer is
therefore checked on sampled output rows: avec_posenet_layer_rows returns the
GPU's own input rows of the layer (the k-row window of every sampled row,
zeros outside the image = the conv's zero padding) and the sampled output
rows; oracle_conv2d_rows recomputes exactly those rows. Fused layers are
checked as executed (pooled outputs via 2x2 max over two conv rows; a fused
pair chains its first layer, bf16-rounded, from the pair's input rows).

Row choice covers the persistent kernels' later passes: tiles are ordered
(branch, image, pixel tile) and strided by the grid, so every row of a later
image (and late rows of every image) is a tile a CTA reaches on its 2nd or
later pass; the last row of an image lies in its (partial) last tile.
"""
from __future__ import annotations

import numpy as np

import oracle_lib as O


def ulp_bf16(x):
    x = np.abs(x).astype(np.float32)
    return np.exp2(np.floor(np.log2(np.maximum(x, 1e-30))) - 7)


def sample_rows(n_img: int, height: int, seed: int, images=None, per_image: int = 2):
    """(image, y) pairs: first and last row of each chosen image plus
    `per_image` seeded random rows, and a few extra rows of the last image."""
    rng = np.random.default_rng(seed)
    if images is None:
        images = range(n_img) if n_img <= 8 else sorted({0, 1, n_img // 2, n_img - 2, n_img - 1,
                                                          *rng.integers(0, n_img, 2).tolist()})
    sel = set()
    for b in images:
        sel.update({(b, 0), (b, height - 1)})
        sel.update((b, int(y)) for y in rng.integers(0, height, per_image))
    last = n_img - 1
    sel.update({(last, 1), (last, height // 2), (last, height - 2)})
    return sorted(sel)


def check_layer_rows(be, h, frame, layers, wb, i, final: bool, seed: int = 0):
    """Compare sampled output rows of conv layer i with the oracle.
    Returns (rel_err, max_abs_err, rows) or None for a layer fused into the next."""
    dims = frame.dims
    kind, src = be.layer_fusion(h, dims, i)
    if kind == 2:  # Mconv6 of a fused head / conv1_1 of conv12: checked through the pair
        return None
    L = layers[i]
    n_img = dims.batch * dims.channels // 3
    ol = be.layer_out_level(h, dims, i)
    pooled = ol > L.level
    hc = dims.height >> L.level  # conv rows at the layer's level
    out_sel = sample_rows(n_img, dims.height >> ol, seed=seed * 1000 + i)
    chain = [src, i] if kind == 3 else [i]
    # rows each conv of the chain must produce, from the last one backwards
    need = [None] * len(chain)
    need[-1] = sorted({(b, 2 * y + d) for b, y in out_sel for d in (0, 1)}) if pooled else list(out_sel)
    for j in range(len(chain) - 1, 0, -1):
        p = layers[chain[j]].k // 2
        need[j - 1] = sorted({(b, y + d) for b, y in need[j] for d in range(-p, p + 1) if 0 <= y + d < hc})
    p0 = layers[chain[0]].k // 2
    in_sel = sorted({(b, y + d) for b, y in need[0] for d in range(-p0, p0 + 1)})
    lin, lout = be.layer_rows(h, frame, i, in_sel, out_sel)
    avail = {r: lin[k] for k, r in enumerate(in_sel)}
    width = lin.shape[1]
    for j, li in enumerate(chain):
        Lj = layers[li]
        p = Lj.k // 2
        cin = Lj.cin
        zero = np.zeros((width, cin), np.float32)
        win = np.stack([np.stack([avail.get((b, y + d), zero) if 0 <= y + d < hc else zero
                                  for d in range(-p, p + 1)]) for b, y in need[j]])
        w, bb, sl = wb[li]
        last = j == len(chain) - 1
        res = O.conv2d_rows(win, w, bb, relu=Lj.act, round_bf16=not (last and final), slope=sl)
        avail = {r: res[k] for k, r in enumerate(need[j])}
    if pooled:
        ref = np.stack([np.maximum(avail[(b, 2 * y)], avail[(b, 2 * y + 1)])
                        .reshape(width // 2, 2, -1).max(axis=1) for b, y in out_sel])
    else:
        ref = np.stack([avail[r] for r in out_sel])
    assert lout.shape == ref.shape, (L.name, lout.shape, ref.shape)
    diff = np.abs(lout - ref)
    err = float(np.linalg.norm(lout - ref) / max(np.linalg.norm(ref), 1e-30))
    assert err <= 1e-3, (L.name, err)
    if not final and kind != 3:  # one rounding: element bound (a chained pair has two)
        tol = ulp_bf16(ref) + 1e-4 * float(np.abs(ref).max())
        bad = diff > tol
        assert not bad.any(), (L.name, int(bad.sum()), float(diff.max()),
                               [out_sel[k] for k in sorted(set(np.nonzero(bad)[0].tolist()))][:8])
    return err, float(diff.max()), len(out_sel)
