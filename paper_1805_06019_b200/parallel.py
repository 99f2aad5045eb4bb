"""Multi-GPU sharding of the full-field decode.

Records are independent per (block location, channel), so a light field
shards by block-row bands with no collective on the data path: each rank
decodes every view restricted to its band.  Bands are balanced by the exact
compressed bytes of each block row (from the offset arrays) plus a constant
per-row pixel cost.  `gather_field` optionally assembles the whole field on
every rank with one NCCL all_gather over NVLink.
"""

import numpy as np


def row_costs(state, bytes_per_pixel_weight=1.0):
    """Per block-row cost: compressed record bytes + output bytes."""
    hdr = state.header
    wb, hb = hdr.block_grid
    cost = np.zeros(hb, dtype=np.float64)
    for c in range(3):
        offs = np.asarray(state.offsets[c], dtype=np.int64)
        ends = np.append(offs[1:], hdr.section_lengths[c][2])
        cost += (ends - offs).reshape(hb, wb).sum(axis=1)
    B = hdr.block_size
    rows_px = np.minimum((np.arange(hb) + 1) * B, hdr.height) - \
        np.arange(hb) * B
    out = rows_px * hdr.width * 3 * hdr.s_count * hdr.t_count
    return cost + bytes_per_pixel_weight * out


def balanced_bands(state, n):
    """n contiguous block-row bands [lo, hi) with near-equal cost."""
    cost = row_costs(state)
    hb = len(cost)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    bounds = [0]
    for k in range(1, n):
        target = cum[-1] * k / n
        b = int(np.searchsorted(cum, target))
        b = min(max(b, bounds[-1]), hb)
        bounds.append(b)
    bounds.append(hb)
    return [(bounds[i], bounds[i + 1]) for i in range(n)]


def gather_field(state, band_out, bands, group=None):
    """All-gather per-rank bands (S, T, rows_r, W, 3) into the full
    (S, T, H, W, 3) field on every rank (NCCL over NVLink)."""
    import torch
    import torch.distributed as dist
    hdr = state.header
    B = hdr.block_size
    rows = [max(0, min(hi * B, hdr.height) - lo * B) for lo, hi in bands]
    pad = max(rows)
    S, T, W = hdr.s_count, hdr.t_count, hdr.width
    send = torch.zeros((S, T, pad, W, 3), dtype=torch.uint8,
                       device=band_out.device)
    send[:, :, :band_out.shape[2]] = band_out
    recv = [torch.empty_like(send) for _ in bands]
    dist.all_gather(recv, send, group=group)
    return torch.cat([r[:, :, :n] for r, n in zip(recv, rows)], dim=2)
