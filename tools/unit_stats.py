"""Dirty-unit statistics of the cfg2 R4 bench stream, recomputed on the host
from the record bitmaps (measurement only): dirty (view, block) units, units
with several present chain levels, units per blend tile (block row, camera
row, 64-pixel chunk)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1805_06019_b200 import container
data, _ = bench.make_stream(bench.CFG)
hdr = container.parse_header(data)
starts, _ = container.section_offsets(hdr)
S, T, h = hdr.s_count, hdr.t_count, hdr.tree_height
wb, hb = hdr.block_grid
nblk = wb * hb
M = sum(container.level_dims(S, T, l)[0] * container.level_dims(S, T, l)[1] for l in range(h))
nbm = (M + 7) // 8
base = {}
b0 = 0
for l in range(h - 1, -1, -1):
    sx, sy = container.level_dims(S, T, l); base[l] = b0; b0 += sx * sy
pres = np.zeros((3, nblk, M), dtype=bool)
for c in range(3):
    off_start = starts[c][1]
    offs = np.frombuffer(data, dtype='<u8', count=nblk, offset=off_start)
    srv0 = starts[c][2]
    idx = srv0 + offs.astype(np.int64)
    raw = np.frombuffer(data, dtype=np.uint8)
    bytes_ = raw[idx[:, None] + np.arange(nbm)[None, :]]
    bits = np.unpackbits(bytes_, axis=1, bitorder='little')[:, :M]
    pres[c] = bits.astype(bool)
# per (t, s) chain presence: per level l node = base[l] + (t>>l)*sx_l + (s>>l)
lev = []
for l in range(h):
    sx, sy = container.level_dims(S, T, l)
    lev.append((l, sx))
units = 0; multi = 0
per_tile = np.zeros((hb, T, wb // 16), dtype=np.int32)
for t in range(T):
    for s in range(S):
        nodes = [base[l] + (t >> l) * sx + (s >> l) for l, sx in lev]
        p = pres[:, :, nodes]            # (3, nblk, h)
        anyp = p.any(axis=(0, 2))        # per block
        nlev = p.any(axis=0).sum(axis=1) # levels present (any channel)
        units += anyp.sum(); multi += (nlev >= 2).sum()
        bi = np.flatnonzero(anyp)
        np.add.at(per_tile, (bi // wb, t, (bi % wb) // 16), 1)
print("dirty units", units, "with >=2 levels", multi, "tiles", per_tile.size)
print("units per tile: mean %.1f p50 %d p90 %d max %d" % (per_tile.mean(), np.median(per_tile), np.percentile(per_tile, 90), per_tile.max()))
