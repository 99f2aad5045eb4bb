"""Native stream producer: synthetic light fields and the .rlfc encoder.

Binds librlfc_producer.so (producer/rlfc_producer.cpp).  Output streams are
byte-identical to the reference encoder's (tests/test_producer.py pins them
against streams the reference produced).  Cluster filter weights and cluster
positions are computed here with numpy exactly as the reference computes them
(hierarchy.py:141-162, 195-212); root views are encoded with Pillow through
container.encode_root, as the reference does (container.py:152-172).
"""

import ctypes
import os

import numpy as np

from . import _build, container
from .errors import FormatError

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.PRODUCER_LIB
        if not os.path.exists(path):
            _build.build_producer()
        L = ctypes.CDLL(path)
        vp, i32, i64, u64 = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                             ctypes.c_uint64)
        L.prod_set_threads.argtypes = [i32]
        L.prod_synthesize.argtypes = [i32, i32, i32, i32, u64, vp]
        L.prod_bise_encode.argtypes = [vp, i64, i32, i32, vp]
        L.prod_bise_encode.restype = i64
        L.prod_encode.argtypes = [i32, i32, i32, i32, vp, i32, i32, i32, i64,
                                  i32, vp]
        L.prod_encode.restype = vp
        L.prod_encode_strip.argtypes = [i32, i32, i32, i32, i32, vp, i32, i32,
                                        i32, i64, i32, vp]
        L.prod_encode_strip.restype = vp
        L.prod_synthesize_rows.argtypes = [i32, i32, i32, i32, u64, i32, i32,
                                           vp]
        L.prod_result_error.argtypes = [vp]
        L.prod_result_srv_len.argtypes = [vp, i32]
        L.prod_result_srv_len.restype = i64
        L.prod_result_copy.argtypes = [vp, i32, vp, vp]
        L.prod_result_roots.argtypes = [vp, vp]
        L.prod_result_present.argtypes = [vp, vp]
        L.prod_free.argtypes = [vp]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def synthesize(spec, threads=0):
    """(S, T, H, W, 3) uint8 of the reference's procedural scene."""
    L = lib()
    L.prod_set_threads(int(threads))
    out = np.empty((spec.s_count, spec.t_count, spec.height, spec.width, 3),
                   dtype=np.uint8)
    L.prod_synthesize(spec.s_count, spec.t_count, spec.width, spec.height,
                      spec.seed & 0xFFFFFFFFFFFFFFFF, _ptr(out))
    return out


def bise_encode(values, rng) -> bytes:
    values = np.ascontiguousarray(values, dtype=np.uint32)
    if values.size and int(values.max()) >= rng.cardinality:
        raise ValueError(
            f"value {int(values.max())} out of range N={rng.cardinality}")
    from .bise import payload_size
    nbits = payload_size(rng, values.size)
    out = np.zeros((nbits + 7) // 8, dtype=np.uint8)
    wrote = lib().prod_bise_encode(_ptr(values), values.size, rng.mode,
                                   rng.low_bits, _ptr(out))
    assert wrote == nbits
    return out.tobytes()


def filter_weights(positions, spec):
    """Integer /256 cluster weights, largest-remainder rounding
    (hierarchy.py:141-162 semantics, numpy float64)."""
    n = len(positions)
    if n == 1:
        return np.array([256], dtype=np.int64)
    if spec.kind == "uniform":
        raw = np.ones(n)
    else:
        pos = np.asarray(positions, dtype=np.float64)
        d2 = ((pos - pos.mean(axis=0)) ** 2).sum(axis=1)
        sig = spec.quantized_sigma()
        raw = np.exp(-d2 / (2.0 * sig * sig))
    scaled = raw * (256 / raw.sum())
    base = np.floor(scaled).astype(np.int64)
    frac = scaled - base
    for i in sorted(range(n), key=lambda i: (-frac[i], i))[:256 - int(base.sum())]:
        base[i] += 1
    return base


def pyramid_weights(camera_positions, tree_height, spec):
    """Flat int64 weights for prod_encode: per level 1..h, per parent (cx
    outer, cy inner), 4 member slots (members x outer, y inner)."""
    pos = np.asarray(camera_positions, dtype=np.float64)
    flat = []
    for _ in range(tree_height):
        sx, sy = pos.shape[:2]
        px, py = -(-sx // 2), -(-sy // 2)
        up = np.zeros((px, py, 2))
        for cx in range(px):
            for cy in range(py):
                members = [(x, y) for x in (2 * cx, 2 * cx + 1) if x < sx
                           for y in (2 * cy, 2 * cy + 1) if y < sy]
                cpos = [pos[x, y] for x, y in members]
                w = filter_weights(cpos, spec)
                slot = np.zeros(4, dtype=np.int64)
                slot[:len(w)] = w
                flat.append(slot)
                up[cx, cy] = (w[:, None] * np.asarray(cpos)).sum(0) / 256.0
        pos = up
    return np.concatenate(flat) if flat else np.zeros(0, np.int64)


def _encode_rows(rgb, S, T, W, h_valid, hp_rows, params, weights):
    """Encode one block-aligned row band: (roots band, [srv_c], [offsets_c],
    present per level)."""
    L = lib()
    B, h = params.block_size, params.tree_height
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    handle = L.prod_encode_strip(S, T, W, h_valid, hp_rows, _ptr(rgb), h, B,
                                 params.pixel_threshold,
                                 params.block_threshold, params.quant_shift,
                                 _ptr(weights))
    try:
        if L.prod_result_error(handle):
            raise FormatError("residual value outside the range table")
        wp = -(-W // B) * B
        nblk = (wp // B) * (hp_rows // B)
        rsx, rsy = container.level_dims(S, T, h)
        roots = np.empty((rsx, rsy, 3, hp_rows, wp), dtype=np.int32)
        L.prod_result_roots(handle, _ptr(roots))
        present = np.zeros(h, dtype=np.int64)
        L.prod_result_present(handle, _ptr(present))
        srvs, offs = [], []
        for c in range(3):
            srv = np.empty(L.prod_result_srv_len(handle, c), dtype=np.uint8)
            off = np.empty(nblk, dtype="<u8")
            L.prod_result_copy(handle, c, _ptr(srv), _ptr(off))
            srvs.append(srv)
            offs.append(off)
    finally:
        L.prod_free(handle)
    return roots, srvs, offs, present


def _assemble(S, T, W, H, params, roots, srvs, offs, present):
    """Root streams + header + sections (container.py:269-339 layout)."""
    from concurrent.futures import ThreadPoolExecutor
    rsx, rsy = container.level_dims(S, T, params.tree_height)
    codec = container.CODEC_IDS[params.root_codec]
    # root planes are coded independently (Pillow releases the GIL while it
    # compresses); the stream order stays channel, y, x
    keys = [(c, y, x) for c in range(3) for y in range(rsy) for x in range(rsx)]

    def one(key):
        c, y, x = key
        return container.encode_root(
            roots[x, y, c].astype(np.int64) + container.CHANNEL_BIAS[c], codec)
    with ThreadPoolExecutor(max_workers=min(len(keys), os.cpu_count() or 1)) as ex:
        blobs = dict(zip(keys, ex.map(one, keys)))
    sections, lengths = [], []
    for c in range(3):
        chunks = []
        for y in range(rsy):
            for x in range(rsx):
                blob = blobs[(c, y, x)]
                chunks.append(len(blob).to_bytes(4, "little"))
                chunks.append(blob)
        root_sec = b"".join(chunks)
        off_sec = np.ascontiguousarray(offs[c], dtype="<u8").tobytes()
        srv_sec = srvs[c].tobytes()
        sections += [root_sec, off_sec, srv_sec]
        lengths.append((len(root_sec), len(off_sec), len(srv_sec)))
    header = container.RlfcHeader(
        s_count=S, t_count=T, width=W, height=H,
        tree_height=params.tree_height, block_size=params.block_size,
        quant_shift=params.quant_shift,
        pixel_threshold=params.pixel_threshold,
        block_threshold=params.block_threshold,
        filter_kind=params.filter.kind,
        sigma_fp=params.filter.sigma_fp if params.filter.kind == "gaussian"
        else 0,
        root_codec_id=codec, section_lengths=tuple(lengths))
    return container.pack_header(header) + b"".join(sections), \
        tuple(int(v) for v in present)


def _encode_rows_gpu(rgb, S, T, W, h_valid, hp_rows, params, weights,
                     device="cuda"):
    """_encode_rows on the GPU (csrc/rlfc_encode.cu): the same outputs --
    (roots band, [srv_c], [offsets_c], present per level) -- from the RKV
    pyramid, the top-down SRV pass with closed-loop reconstruction and the
    record serialisation run as CUDA kernels."""
    import torch
    from . import _native
    L = _native.lib()
    dev = torch.device(device)
    B, h = params.block_size, params.tree_height
    bsq = B * B
    wp = -(-W // B) * B
    hp = hp_rows
    wb, hb = wp // B, hp // B
    nblk = wb * hb
    plane = hp * wp
    ldim = lambda n, l: -(-n // (1 << l))                          # noqa: E731
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        d_rgb = torch.from_numpy(np.ascontiguousarray(rgb, dtype=np.uint8)).to(dev)
        lv = [torch.empty(S * T * 3 * plane, dtype=torch.int32, device=dev)]
        _native.check(L.rlfc_enc_planes(d_rgb.data_ptr(), S * T, W, h_valid, hp, wp, lv[0].data_ptr(), stream),
                      "rlfc_enc_planes")
        del d_rgb
        d_w = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.int64)).to(dev)
        woff = 0
        for l in range(1, h + 1):
            sx, sy, px, py = ldim(S, l - 1), ldim(T, l - 1), ldim(S, l), ldim(T, l)
            lv.append(torch.empty(px * py * 3 * plane, dtype=torch.int32, device=dev))
            _native.check(L.rlfc_enc_pyramid(lv[l - 1].data_ptr(), sx, sy, lv[l].data_ptr(), px, py,
                                             d_w.data_ptr() + 8 * woff, hp, wp, stream), "rlfc_enc_pyramid")
            woff += px * py * 4
        rsx, rsy = ldim(S, h), ldim(T, h)
        roots = lv[h].view(rsx, rsy, 3, hp, wp).cpu().numpy()
        base, M = {}, 0
        for l in range(h - 1, -1, -1):
            base[l] = M
            M += ldim(S, l) * ldim(T, l)
        desc = torch.full((3 * nblk * M,), 0xFF, dtype=torch.uint8, device=dev)
        zv = torch.empty(3 * nblk * M * bsq, dtype=torch.int16, device=dev)
        present = torch.zeros(h, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        above = lv[h]
        for l in range(h - 1, -1, -1):
            sx, sy, psy = ldim(S, l), ldim(T, l), ldim(T, l + 1)
            _native.check(L.rlfc_enc_srv_level(
                lv[l].data_ptr(), above.data_ptr(), sx, sy, psy, hp, wp, B, params.pixel_threshold,
                params.block_threshold, params.quant_shift, base[l], M, desc.data_ptr(), zv.data_ptr(),
                present.data_ptr() + 8 * l, err.data_ptr(), stream), "rlfc_enc_srv_level")
            above = lv[l]
        if err.item():
            raise FormatError("residual value outside the range table")
        nrec = 3 * nblk
        size = torch.empty(nrec, dtype=torch.int64, device=dev)
        _native.check(L.rlfc_enc_record_sizes(desc.data_ptr(), nrec, M, bsq, size.data_ptr(), stream),
                      "rlfc_enc_record_sizes")
        ends = torch.cumsum(size, 0)
        starts = ends - size
        total = int(ends[-1].item()) if nrec else 0
        out = torch.empty(max(1, total), dtype=torch.uint8, device=dev)
        _native.check(L.rlfc_enc_records(desc.data_ptr(), zv.data_ptr(), nrec, M, bsq, starts.data_ptr(),
                                         out.data_ptr(), stream), "rlfc_enc_records")
        starts_h = starts.cpu().numpy()
        out_h = out.cpu().numpy()
        srvs, offs = [], []
        for c in range(3):
            c0 = int(starts_h[c * nblk]) if nblk else 0
            c1 = int(starts_h[(c + 1) * nblk]) if c < 2 else total
            offs.append((starts_h[c * nblk:(c + 1) * nblk] - c0).astype("<u8"))
            srvs.append(out_h[c0:c1].copy())
        return roots.astype(np.int32), srvs, offs, present.cpu().numpy()


def encode_gpu(lf, params, device="cuda"):
    """encode() with the RKV/SRV trees and the records built on the GPU;
    root views are still coded by Pillow on the host (container.py:152-172)."""
    S, T, W, H = lf.s_count, lf.t_count, lf.width, lf.height
    w = np.ascontiguousarray(pyramid_weights(lf.camera_positions,
                                             params.tree_height, params.filter))
    hp = -(-H // params.block_size) * params.block_size
    roots, srvs, offs, present = _encode_rows_gpu(lf.rgb, S, T, W, H, hp, params, w, device)
    return _assemble(S, T, W, H, params, roots, srvs, offs, present)


def encode(lf, params, threads=0):
    """(stream bytes, present blocks per level) for a LightFieldGrid."""
    lib().prod_set_threads(int(threads))
    S, T, W, H = lf.s_count, lf.t_count, lf.width, lf.height
    w = np.ascontiguousarray(pyramid_weights(lf.camera_positions,
                                             params.tree_height, params.filter))
    hp = -(-H // params.block_size) * params.block_size
    roots, srvs, offs, present = _encode_rows(lf.rgb, S, T, W, H, hp, params,
                                              w)
    return _assemble(S, T, W, H, params, roots, srvs, offs, present)


def encode_synthetic_striped(spec, params, strip_rows=64, threads=0):
    """Synthesise and encode a large synthetic field band by band.

    Every RKV/SRV operation is per pixel or per block (hierarchy.py:182-271)
    and records are per block (container.py:306-323), so encoding
    block-aligned row bands independently and stitching the records, offsets
    and root rows reproduces the monolithic stream byte for byte
    (tests/test_producer.py).  Peak memory is one band, which makes the
    32x32x2048^2 configuration (12.9 GB of RGB) feasible.
    """
    from .lightfield import grid_positions
    L = lib()
    L.prod_set_threads(int(threads))
    S, T, W, H = spec.s_count, spec.t_count, spec.width, spec.height
    B, h = params.block_size, params.tree_height
    strip_rows = max(B, strip_rows // B * B)
    hp = -(-H // B) * B
    wp = -(-W // B) * B
    w = np.ascontiguousarray(pyramid_weights(grid_positions(S, T), h,
                                             params.filter))
    rsx, rsy = container.level_dims(S, T, h)
    roots = np.empty((rsx, rsy, 3, hp, wp), dtype=np.int32)
    srv_parts = [[], [], []]
    off_parts = [[], [], []]
    base = [0, 0, 0]
    present = np.zeros(h, dtype=np.int64)
    for y0 in range(0, hp, strip_rows):
        y1 = min(y0 + strip_rows, hp)
        valid = max(0, min(y1, H) - y0)
        rgb = np.empty((S, T, valid, W, 3), dtype=np.uint8)
        if valid:
            L.prod_synthesize_rows(S, T, W, H, spec.seed & 0xFFFFFFFFFFFFFFFF,
                                   y0, y0 + valid, _ptr(rgb))
        r, srvs, offs, pres = _encode_rows(rgb, S, T, W, valid, y1 - y0,
                                           params, w)
        roots[:, :, :, y0:y1] = r
        present += pres
        for c in range(3):
            off_parts[c].append(offs[c] + np.uint64(base[c]))
            srv_parts[c].append(srvs[c])
            base[c] += len(srvs[c])
    srvs = [np.concatenate(p) for p in srv_parts]
    offs = [np.concatenate(p) for p in off_parts]
    return _assemble(S, T, W, H, params, roots, srvs, offs, present)
