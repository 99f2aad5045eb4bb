"""Reversible integer YCoCg-R lifting (host-side helpers).

Same arithmetic as the reference colorspace.py:15-56 (floor half-shifts,
clamped inverse).  The decode kernels fuse the inverse transform into their
epilogue; these numpy helpers serve the producer, metrics and tests.
"""

import numpy as np

CHROMA_BIAS = 256


def rgb_to_ycocgr(r, g, b):
    r, g, b = (np.asarray(v, dtype=np.int32) for v in (r, g, b))
    co = r - b
    tmp = b + (co >> 1)
    cg = g - tmp
    return tmp + (cg >> 1), co, cg


def ycocgr_to_rgb(y, co, cg):
    y, co, cg = (np.asarray(v, dtype=np.int32) for v in (y, co, cg))
    tmp = y - (cg >> 1)
    b = tmp - (co >> 1)
    return b + co, cg + tmp, b


def grid_to_planes(rgb):
    rgb = np.asarray(rgb)
    return list(rgb_to_ycocgr(rgb[..., 0], rgb[..., 1], rgb[..., 2]))


def planes_to_grid(planes, clamp=True):
    rgb = np.stack(ycocgr_to_rgb(*planes), axis=-1)
    if clamp:
        rgb = np.clip(rgb, 0, 255)
    return rgb.astype(np.uint8)
