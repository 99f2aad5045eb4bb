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


def band_rows(state, bands):
    """Pixel rows of each block-row band."""
    B, H = state.header.block_size, state.header.height
    return [max(0, min(hi * B, H) - lo * B) for lo, hi in bands]


def gather_field(state, band_out, bands, group=None):
    """All-gather every rank's band (S, T, rows_r, W, 3) into one band-major
    tensor (n_bands, S, T, rows_max, W, 3) on every rank: one
    all_gather_into_tensor (NCCL over NVLink between GPUs), no concatenation
    copy.  Bands shorter than the longest are padded (only the short ones
    are copied); band_major_to_grid gives the (S, T, H, W, 3) layout."""
    import torch
    import torch.distributed as dist
    hdr = state.header
    rows = band_rows(state, bands)
    pad = max(rows)
    S, T, W = hdr.s_count, hdr.t_count, hdr.width
    if band_out.shape[2] == pad and band_out.is_contiguous():
        send = band_out
    else:
        send = torch.zeros((S, T, pad, W, 3), dtype=torch.uint8, device=band_out.device)
        send[:, :, :band_out.shape[2]] = band_out
    recv = torch.empty(len(bands) * send.numel(), dtype=torch.uint8, device=band_out.device)
    dist.all_gather_into_tensor(recv, send.reshape(-1), group=group)
    return recv.view(len(bands), S, T, pad, W, 3)


def band_major_to_grid(recv, state, bands):
    """(S, T, H, W, 3) copy of a band-major gather (the reference decode_all
    layout)."""
    import torch
    rows = band_rows(state, bands)
    return torch.cat([recv[i, :, :, :n] for i, n in enumerate(rows)], dim=2)
