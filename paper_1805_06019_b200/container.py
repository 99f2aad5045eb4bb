"""Stream container: header, sections, BFS node geometry, random-access locate.

The wire format is the reference's, unchanged (reference container.py:1-27,
SPEC.md:381-403):

    header (64 bytes, little-endian)
    per channel (Y, Co, Cg):
        root stream   per root view (y outer, x inner): u32 length + blob
        offset array  u64 per spatial block, relative to the SRV stream
        SRV stream    one record per spatial block, row-major

Everything here is host-side, init-time parsing; the per-block work runs on
the GPU (decoder.py).
"""

import io
import os
import struct
import threading
from dataclasses import dataclass

import numpy as np

from .bise import RANGE_TABLE, payload_bytes_table
from .errors import FormatError, UnsupportedCodecError

MAGIC = b"RLFC"
VERSION = 1
HEADER_SIZE = 64
HEADER_FORMAT = "<4sBBBBHHHHBBHHI2x9I"     # container.py:46
assert struct.calcsize(HEADER_FORMAT) == HEADER_SIZE

CODEC_RAW, CODEC_PNG, CODEC_JPEG2000 = 0, 1, 2
CODEC_IDS = {"raw": CODEC_RAW, "png": CODEC_PNG, "jpeg2000": CODEC_JPEG2000}
CODEC_NAMES = {v: k for k, v in CODEC_IDS.items()}
FILTER_IDS = {"uniform": 0, "gaussian": 1}
FILTER_NAMES = {v: k for k, v in FILTER_IDS.items()}
VALID_BLOCK_SIZES = (2, 4, 8, 16)
CHANNEL_BIAS = (0, 256, 256)


def padded_dims(width, height, block_size):
    return -(-width // block_size) * block_size, \
        -(-height // block_size) * block_size


@dataclass(frozen=True)
class RlfcHeader:
    """Decoded 64-byte header (fields as reference container.py:59-95)."""
    s_count: int
    t_count: int
    width: int
    height: int
    tree_height: int
    block_size: int
    quant_shift: int
    pixel_threshold: int
    block_threshold: int
    filter_kind: str
    sigma_fp: int
    root_codec_id: int
    section_lengths: tuple

    @property
    def padded_dims(self):
        return padded_dims(self.width, self.height, self.block_size)

    @property
    def block_grid(self):
        wp, hp = self.padded_dims
        return wp // self.block_size, hp // self.block_size

    def params(self):
        from .encoder import EncodingParams, FilterSpec
        sigma = self.sigma_fp / 256.0 if self.filter_kind == "gaussian" \
            else 0.7
        return EncodingParams(
            tree_height=self.tree_height, block_size=self.block_size,
            pixel_threshold=self.pixel_threshold,
            block_threshold=self.block_threshold,
            quant_shift=self.quant_shift,
            filter=FilterSpec(kind=self.filter_kind, sigma=sigma),
            root_codec=CODEC_NAMES[self.root_codec_id])


# --- BFS tree geometry (container.py:102-145) --------------------------------

def level_dims(s_count, t_count, level):
    """Camera-grid dims at a tree level: repeated ceil-halving."""
    return -(-s_count >> level), -(-t_count >> level)


def level_node_counts(s_count, t_count, tree_height):
    return [level_dims(s_count, t_count, l)[0] *
            level_dims(s_count, t_count, l)[1] for l in range(tree_height)]


def total_srv_nodes(s_count, t_count, tree_height):
    return int(sum(level_node_counts(s_count, t_count, tree_height)))


def level_bases(s_count, t_count, tree_height):
    """Serial index of the first node of each level (level h-1 is first)."""
    counts = level_node_counts(s_count, t_count, tree_height)
    bases, acc = [0] * tree_height, 0
    for l in range(tree_height - 1, -1, -1):
        bases[l] = acc
        acc += counts[l]
    return bases


def bfs_index(level, x, y, s_count, t_count, tree_height):
    if not 0 <= level < tree_height:
        raise ValueError(f"level {level} outside SRV tree")
    sx, sy = level_dims(s_count, t_count, level)
    if not (0 <= x < sx and 0 <= y < sy):
        raise ValueError(f"node ({x}, {y}) outside level-{level} grid")
    return level_bases(s_count, t_count, tree_height)[level] + y * sx + x


def ancestors(s, t, s_count, t_count, tree_height):
    """[(level, x, y)] from level h-1 down to 0, plus the root cell."""
    if not (0 <= s < s_count and 0 <= t < t_count):
        raise ValueError(f"image index ({s}, {t}) outside grid")
    return ([(l, s >> l, t >> l) for l in range(tree_height - 1, -1, -1)],
            (s >> tree_height, t >> tree_height))


def chain_node_indices(s, t, s_count, t_count, tree_height):
    chain, _ = ancestors(s, t, s_count, t_count, tree_height)
    return np.asarray([bfs_index(l, x, y, s_count, t_count, tree_height)
                       for l, x, y in chain], dtype=np.int64)


def all_chains(s_count, t_count, tree_height):
    """chains[s, t, :] for every image, vectorised (decoder.py:40-44)."""
    bases = level_bases(s_count, t_count, tree_height)
    s = np.arange(s_count)[:, None, None]
    t = np.arange(t_count)[None, :, None]
    lv = np.arange(tree_height - 1, -1, -1)[None, None, :]
    sx = np.array([level_dims(s_count, t_count, l)[0]
                   for l in range(tree_height)])
    base = np.array(bases)
    return (base[lv] + (t >> lv) * sx[lv] + (s >> lv)).astype(np.int64)


# --- header -------------------------------------------------------------------

def pack_header(header: RlfcHeader) -> bytes:
    flat = [int(v) for sec in header.section_lengths for v in sec]
    return struct.pack(
        HEADER_FORMAT, MAGIC, VERSION, header.root_codec_id,
        header.block_size, header.tree_height, header.s_count,
        header.t_count, header.width, header.height, header.quant_shift,
        FILTER_IDS[header.filter_kind], header.sigma_fp,
        header.pixel_threshold, header.block_threshold, *flat)


def parse_header(data) -> RlfcHeader:
    """Validate and decode the header (same checks as container.py:214-243)."""
    if len(data) < HEADER_SIZE:
        raise FormatError(f"stream too short for header: {len(data)} bytes")
    (magic, version, codec, block, height_tree, s_count, t_count, width,
     height, shift, filt, sigma_fp, p_thr, b_thr, *flat) = struct.unpack(
        HEADER_FORMAT, bytes(data[:HEADER_SIZE]))
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}")
    if version != VERSION:
        raise FormatError(f"unsupported version {version}")
    if codec not in CODEC_NAMES:
        raise UnsupportedCodecError(f"unknown root codec id {codec}")
    if block not in VALID_BLOCK_SIZES:
        raise FormatError(f"invalid block size {block}")
    if height_tree < 1:
        raise FormatError("tree height must be >= 1")
    if filt not in FILTER_NAMES:
        raise FormatError(f"invalid filter kind {filt}")
    if min(s_count, t_count, width, height) < 1:
        raise FormatError("grid and image dims must be >= 1")
    return RlfcHeader(
        s_count=s_count, t_count=t_count, width=width, height=height,
        tree_height=height_tree, block_size=block, quant_shift=shift,
        pixel_threshold=p_thr, block_threshold=b_thr,
        filter_kind=FILTER_NAMES[filt], sigma_fp=sigma_fp,
        root_codec_id=codec,
        section_lengths=tuple(tuple(flat[3 * c:3 * c + 3]) for c in range(3)))


def section_offsets(header: RlfcHeader):
    """Absolute (root, offsets, srv) starts per channel, and the stream end."""
    starts, pos = [], HEADER_SIZE
    for root_len, off_len, srv_len in header.section_lengths:
        starts.append((pos, pos + root_len, pos + root_len + off_len))
        pos += root_len + off_len + srv_len
    return starts, pos


def check_stream_length(header: RlfcHeader, data):
    _, end = section_offsets(header)
    if len(data) < end:
        raise FormatError(f"stream truncated: {len(data)} < {end} bytes")
    if len(data) > end:
        raise FormatError(
            f"{len(data) - end} trailing bytes after the last section")


# --- root views -----------------------------------------------------------------

def decode_root(blob, codec_id, width, height):
    """One lossless 16-bit root plane (container.py:175-195 semantics)."""
    if codec_id == CODEC_RAW:
        if len(blob) != width * height * 2:
            raise FormatError(
                f"raw root length {len(blob)} != {width * height * 2}")
        return np.frombuffer(blob, dtype="<u2").reshape(height, width) \
            .astype(np.int64)
    if codec_id in (CODEC_PNG, CODEC_JPEG2000):
        from PIL import Image
        try:
            with Image.open(io.BytesIO(blob)) as im:
                arr = np.asarray(im)
        except Exception as exc:
            raise FormatError(f"root image decode failed: {exc}") from exc
        if arr.ndim != 2:
            raise FormatError("root image is not single-channel")
        if arr.shape != (height, width):
            raise FormatError(
                f"root dims {arr.shape[::-1]} != header {(width, height)}")
        return arr.astype(np.int64)
    raise UnsupportedCodecError(f"unknown root codec id {codec_id}")


def encode_root(plane, codec_id) -> bytes:
    arr = np.asarray(plane)
    if arr.min() < 0 or arr.max() > 0xFFFF:
        raise ValueError("root plane out of unsigned 16-bit range")
    arr = arr.astype(np.uint16)
    if codec_id == CODEC_RAW:
        return arr.astype("<u2").tobytes()
    from PIL import Image
    buf = io.BytesIO()
    if codec_id == CODEC_PNG:
        Image.fromarray(arr).save(buf, format="PNG")
    elif codec_id == CODEC_JPEG2000:
        try:
            Image.fromarray(arr).save(buf, format="JPEG2000",
                                      irreversible=False)
        except Exception as exc:
            raise UnsupportedCodecError(
                f"jpeg2000 encoding unavailable: {exc}") from exc
    else:
        raise UnsupportedCodecError(f"unknown root codec id {codec_id}")
    return buf.getvalue()


def parse_roots(data, header: RlfcHeader, threads=None):
    """All root planes, (rsx, rsy, 3, Hp, Wp) int32 with the bias removed.

    The section layout is walked serially (container.py:355-379); the plane
    images, Pillow decodes that release the GIL, are decoded on a thread pool.
    The first failure in stream order is raised, exactly as the reference's
    plane-by-plane loop meets it: a decode error of an earlier plane before a
    truncation or trailing bytes found later.
    """
    from concurrent.futures import ThreadPoolExecutor
    wp, hp = header.padded_dims
    rsx, rsy = level_dims(header.s_count, header.t_count, header.tree_height)
    starts, _ = section_offsets(header)
    out = np.zeros((rsx, rsy, 3, hp, wp), dtype=np.int32)
    events = []            # ("plane", (x, y, c), blob) | ("error", exc)
    for c in range(3):
        pos = starts[c][0]
        end = pos + header.section_lengths[c][0]
        stop = False
        for y in range(rsy):
            for x in range(rsx):
                if pos + 4 > end or pos + 4 + struct.unpack_from("<I", data, pos)[0] > end:
                    events.append(("error", FormatError("root stream truncated")))
                    stop = True
                    break
                (n,) = struct.unpack_from("<I", data, pos)
                pos += 4
                events.append(("plane", (x, y, c), bytes(data[pos:pos + n])))
                pos += n
            if stop:
                break
        if stop:
            break
        if pos != end:
            events.append(("error", FormatError("trailing bytes in root stream")))
            break
    planes = [e for e in events if e[0] == "plane"]

    def dec(e):
        try:
            return decode_root(e[2], header.root_codec_id, wp, hp), None
        except Exception as exc:          # raised below in stream order
            return None, exc

    nthreads = threads or min(32, os.cpu_count() or 1)
    if header.root_codec_id == CODEC_RAW or nthreads <= 1 or len(planes) <= 1:
        results = [dec(e) for e in planes]
    else:
        with ThreadPoolExecutor(max_workers=nthreads) as ex:
            results = list(ex.map(dec, planes))
    it = iter(results)
    for e in events:
        if e[0] == "error":
            raise e[1]
        arr, exc = next(it)
        if exc is not None:
            raise exc
        x, y, c = e[1]
        out[x, y, c] = arr - CHANNEL_BIAS[c]
    return out


_PNG_SIG = b"\x89PNG\r\n\x1a\n"


def _png_idat(blob, width, height):
    """The zlib stream of a 16-bit greyscale, non-interlaced PNG of the
    header's dims with valid chunk CRCs, or None (anything else goes to
    Pillow, which raises the reference's errors)."""
    import zlib
    if blob[:8] != _PNG_SIG:
        return None
    pos, idat, seen_end, ihdr_ok = 8, [], False, False
    while pos + 12 <= len(blob):
        (n,) = struct.unpack_from(">I", blob, pos)
        typ = blob[pos + 4:pos + 8]
        if pos + 12 + n > len(blob):
            return None
        body = blob[pos + 8:pos + 8 + n]
        if zlib.crc32(typ + body) != struct.unpack_from(">I", blob, pos + 8 + n)[0]:
            return None
        if typ == b"IHDR":
            if n != 13 or struct.unpack(">IIBBBBB", body) != (width, height, 16, 0, 0, 0, 0):
                return None
            ihdr_ok = True
        elif typ == b"IDAT":
            idat.append(body)
        elif typ == b"IEND":
            seen_end = True
            break
        elif typ[0] & 0x20 == 0:            # unknown critical chunk
            return None
        pos += 12 + n
    if not (ihdr_ok and seen_end and idat):
        return None
    return b"".join(idat)


_POOL = None
_POOL_LOCK = threading.Lock()


def _inflate_pool():
    """Process-wide thread pool for the root-view inflates (zlib releases
    the GIL); created once, so an init does not pay thread start-up."""
    global _POOL
    from concurrent.futures import ThreadPoolExecutor
    with _POOL_LOCK:
        if _POOL is None:
            _POOL = ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1),
                                       thread_name_prefix="rlfc-inflate")
        return _POOL


def parse_roots_device(data, header: RlfcHeader, device, threads=None):
    """Root planes decoded on the GPU (container.py:175-195; PNG and RAW roots):
    the host walks the sections and inflates each plane's IDAT stream on a
    thread pool; the PNG scanline filters are undone by rlfc_png_unfilter
    and the channel bias removed by rlfc_root_planes straight into the
    device root tensor (rsx, rsy, 3, Hp, Wp) (int16 when every sample fits,
    else int32).  Returns the device tensor, or None when
    the stream is not a plain 16-bit PNG-root stream; the caller then takes
    parse_roots (Pillow), which raises exactly the reference's errors."""
    import zlib
    from concurrent.futures import ThreadPoolExecutor
    import torch
    from . import _native
    if header.root_codec_id not in (CODEC_PNG, CODEC_RAW):
        return None
    wp, hp = header.padded_dims
    rsx, rsy = level_dims(header.s_count, header.t_count, header.tree_height)
    starts, _ = section_offsets(header)
    spans = []
    for c in range(3):
        pos = starts[c][0]
        end = pos + header.section_lengths[c][0]
        for _ in range(rsy * rsx):
            if pos + 4 > end:
                return None
            (n,) = struct.unpack_from("<I", data, pos)
            if pos + 4 + n > end:
                return None
            spans.append((pos + 4, n))
            pos += 4 + n
        if pos != end:
            return None
    L = _native.lib()
    dev = torch.device(device)
    if header.root_codec_id == CODEC_RAW:
        # little-endian 16-bit samples as stored (container.py:175-195): one
        # pinned copy, one upload, the bias removed on the device
        if any(n != wp * hp * 2 for _, n in spans):
            return None                    # decode_root raises the reference's error
        host = torch.empty((len(spans), hp * wp), dtype=torch.int16).pin_memory()
        hv = host.numpy().view(np.uint8).reshape(len(spans), -1)
        mv = memoryview(data)
        for i, (a, n) in enumerate(spans):
            hv[i] = np.frombuffer(mv[a:a + n], dtype=np.uint8)
        with torch.cuda.device(dev):
            samples = host.to(dev, non_blocking=True)
        return _root_planes_device(L, samples, len(spans), rsx, rsy, hp, wp, dev)
    blobs = [bytes(data[a:a + n]) for a, n in spans]
    stride = hp * (1 + 2 * wp)

    def inflate(b):
        z = _png_idat(b, wp, hp)
        if z is None:
            return None
        try:
            raw = zlib.decompress(z)
        except zlib.error:
            return None
        return raw if len(raw) == stride else None

    if threads:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            raws = list(ex.map(inflate, blobs))
    else:
        raws = list(_inflate_pool().map(inflate, blobs))
    if any(r is None for r in raws):
        return None
    host = torch.empty((len(raws), stride), dtype=torch.uint8).pin_memory()
    hv = host.numpy()
    for i, r in enumerate(raws):
        hv[i] = np.frombuffer(r, dtype=np.uint8)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        raw_d = host.to(dev, non_blocking=True)
        samples = torch.empty((len(raws), hp, wp), dtype=torch.int16, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        _native.check(L.rlfc_png_unfilter(raw_d.data_ptr(), stride, len(raws), wp, hp, samples.data_ptr(),
                                          hp * wp, bad.data_ptr(), stream), "rlfc_png_unfilter")
        if bad.item():
            return None
    return _root_planes_device(L, samples, len(raws), rsx, rsy, hp, wp, dev)


def _root_planes_device(L, samples, nplanes, rsx, rsy, hp, wp, dev):
    """Bias removal + scatter into the (rsx, rsy, 3, Hp, Wp) root tensor
    (rlfc_root_planes): int16 when every sample fits, else int32."""
    import torch
    from . import _native
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        roots = torch.empty((rsx, rsy, 3, hp, wp), dtype=torch.int16, device=dev)
        mm = torch.tensor([1 << 30, -(1 << 30)], dtype=torch.int32, device=dev)
        _native.check(L.rlfc_root_planes(samples.data_ptr(), nplanes, rsx, rsy, hp, wp, 1, roots.data_ptr(),
                                         mm.data_ptr(), stream), "rlfc_root_planes")
        lo, hi = mm.cpu().tolist()
        if lo < -32768 or hi > 32767:
            roots = torch.empty((rsx, rsy, 3, hp, wp), dtype=torch.int32, device=dev)
            _native.check(L.rlfc_root_planes(samples.data_ptr(), nplanes, rsx, rsy, hp, wp, 0, roots.data_ptr(),
                                             None, stream), "rlfc_root_planes")
    return roots


def parse_offsets(data, header: RlfcHeader, channel):
    wb, hb = header.block_grid
    starts, _ = section_offsets(header)
    length = header.section_lengths[channel][1]
    if length != wb * hb * 8:
        raise FormatError(f"offset array length {length} != {wb * hb * 8}")
    return np.frombuffer(data, dtype="<u8", count=wb * hb,
                         offset=starts[channel][1])


def srv_section(data, header: RlfcHeader, channel):
    starts, _ = section_offsets(header)
    return np.frombuffer(data, dtype=np.uint8,
                         count=header.section_lengths[channel][2],
                         offset=starts[channel][2])


def locate_block(data, header: RlfcHeader, channel, blk_index, node_index):
    """(payload_start, payload_end, descriptor) of one node, or None.

    Host-side random-access locate (container.py:402-445 semantics): touches
    the record's bitmap and the descriptors of earlier present nodes only.
    """
    wb, hb = header.block_grid
    if not 0 <= blk_index < wb * hb:
        raise ValueError(f"block index {blk_index} outside grid")
    m = total_srv_nodes(header.s_count, header.t_count, header.tree_height)
    if not 0 <= node_index < m:
        raise ValueError(f"node index {node_index} outside tree")
    starts, _ = section_offsets(header)
    srv_start = starts[channel][2]
    srv_end = srv_start + header.section_lengths[channel][2]
    rec = srv_start + int(parse_offsets(data, header, channel)[blk_index])
    nbm = (m + 7) >> 3
    if rec + nbm > srv_end:
        raise FormatError("record offset past section end")
    bitmap = np.unpackbits(np.frombuffer(bytes(data[rec:rec + nbm]),
                                         np.uint8), bitorder="little")
    if not bitmap[node_index]:
        return None
    pbytes = payload_bytes_table(header.block_size ** 2)
    cursor = rec + nbm
    for node in np.flatnonzero(bitmap[:node_index + 1]):
        if cursor >= srv_end:
            raise FormatError("record truncated mid-scan")
        desc = data[cursor]
        if desc >= len(RANGE_TABLE):
            raise FormatError(f"descriptor {desc} outside range table")
        if node == node_index:
            end = cursor + 1 + int(pbytes[desc])
            if end > srv_end:
                raise FormatError("payload past section end")
            return cursor + 1, end, desc
        cursor += 1 + int(pbytes[desc])
    raise AssertionError("unreachable")
