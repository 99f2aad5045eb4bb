"""Stream decoding on the B200: drop-in for the reference rlfc.decoder.

Public functions keep the reference signatures, return types and exceptions
(reference decoder.py:31-210): `init`, `decode_block_progressive`,
`decode_block`, `decode_block_traced`, `decode_plane`, `decode_image`,
`decode_all`.  `init` parses the header and root views on the host exactly
once and uploads the SRV sections, offset arrays and root planes to HBM; every
decode afterwards is a CUDA kernel from librlfc_b200.so (include/rlfc_b200.h).

The batched, device-resident API used for throughput work is
`decode_field` (whole light field or any image subset / block-row band,
returned as a CUDA tensor), `decode_blocks` (random-access batches),
`decode_planes` and `bise_decode_batch`.

There is no CPU fallback: without the extension or a CUDA device these
functions raise `_native.NativeUnavailable`.
"""

import ctypes
import os
import struct
import threading
import weakref
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native, colorspace, container
from .bise import RANGE_TABLE, payload_bytes_table
from .errors import FormatError
from .lightfield import LightFieldGrid, default_geometry, grid_positions

# zero bytes after each device SRV section: 64-bit bit windows read up to 8
# bytes past a payload, and the single-block kernel stages whole 16-byte
# lines up to 31 bytes past the record end
SRV_TAIL_PAD = 32


def _torch():
    import torch
    return torch


def _host_bytes(arr):
    """A CPU uint8 tensor viewing a (possibly read-only) host byte array
    without copying it; only ever read (the source of an upload)."""
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return _torch().from_numpy(np.asarray(arr, dtype=np.uint8).reshape(-1))


_cuda_get_device = None


def _get_device():
    """The calling thread's current CUDA device index (CUDA initialised)."""
    global _cuda_get_device
    if _cuda_get_device is None:
        _cuda_get_device = _torch()._C._cuda_getDevice
    return _cuda_get_device()


def _field_on(state, device=None):
    """state.device_field(device) without its lock and device object when
    the field of the current device is already uploaded (a dict read is
    atomic; a field exists only once CUDA is initialised)."""
    if device is None and state._devices:
        df = state._devices.get(_get_device())
        if df is not None:
            return df
    return state.device_field(device)


class DeviceField:
    """One stream resident in one GPU's HBM plus its `rlfc_field` descriptor.

    Layout: per channel the SRV section as
    raw bytes (+16 zero bytes so 8-byte bit-window loads never leave the
    allocation) and the u64 offset array; the root planes as one
    (rsx, rsy, 3, Hp, Wp) int16 tensor (int32 if any sample needs it).
    """

    def __init__(self, header, srv, offsets, root_planes, device, roots_dev=None):
        torch = _torch()
        self.device = torch.device(device)
        self.header = header
        S, T, h = header.s_count, header.t_count, header.tree_height
        if h > _native.MAX_LEVELS:
            raise FormatError(f"tree height {h} above the supported "
                              f"{_native.MAX_LEVELS} levels")
        self.srv = []
        self.offsets = []
        for c in range(3):
            # straight from the stream bytes into HBM (no host copies of the
            # section), then the zero tail on the device
            n = len(srv[c])
            buf = torch.empty(n + SRV_TAIL_PAD, dtype=torch.uint8, device=self.device)
            buf[n:].zero_()
            if n:
                buf[:n].copy_(_host_bytes(srv[c]))
            self.srv.append(buf)
            off = np.ascontiguousarray(offsets[c]).view(np.int64)
            self.offsets.append(torch.from_numpy(off.copy()).to(self.device))
        if roots_dev is not None and roots_dev.device == self.device:
            # decoded on this GPU at init (container.parse_roots_device)
            self.roots = roots_dev
            i16 = roots_dev.dtype == torch.int16
        else:
            i16 = bool(root_planes.size == 0 or (root_planes.min() >= -32768 and
                                                 root_planes.max() <= 32767))
            rp = root_planes.astype(np.int16 if i16 else np.int32)
            self.roots = torch.from_numpy(np.ascontiguousarray(rp)).to(self.device)
        f = _native.RlfcField()
        wp, hp = header.padded_dims
        wb, hb = header.block_grid
        rsx, rsy = container.level_dims(S, T, h)
        m = container.total_srv_nodes(S, T, h)
        f.s_count, f.t_count, f.width, f.height = S, T, header.width, \
            header.height
        f.block, f.tree_height, f.quant_shift = header.block_size, h, \
            header.quant_shift
        f.m_nodes, f.wp, f.hp, f.wb, f.hb, f.rsx, f.rsy = m, wp, hp, wb, hb, \
            rsx, rsy
        f.roots_i16 = int(i16)
        f.bitmap_bytes = (m + 7) >> 3
        for l, base in enumerate(container.level_bases(S, T, h)):
            f.level_base[l] = base
            f.level_sx[l], f.level_sy[l] = container.level_dims(S, T, l)
        for c in range(3):
            f.srv[c] = self.srv[c].data_ptr()
            f.offsets[c] = self.offsets[c].data_ptr()
            f.srv_len[c] = len(srv[c])
        f.roots = self.roots.data_ptr()
        f.tile_bytes_max = tile_bytes_max(header, offsets)
        self.cfield = f
        self.ref = ctypes.byref(f)
        self._ws_lock = threading.Lock()
        # the staged path's workspace is shared by every caller enqueueing on
        # the same CUDA stream: its whole launch sequence is enqueued under
        # this lock so two threads' sequences never interleave
        self.enqueue_lock = threading.Lock()
        self._ws = {}
        self._ws_bytes = 0
        self._present = None
        self._dir = None
        self.block_scratch = {}      # thread id -> _BlockScratch
        self._index_view = None      # rlfc_index_view (index_view()), False: none
        self.render_field = None     # renderer's tap-camera scratch (under enqueue_lock)

    def directory(self):
        """The device record directory (rlfc_b200.h rlfc_dir: tile-major
        payload blobs, blob offsets, root colours, anomaly list), built on
        the GPU on first use; None outside its envelope."""
        torch = _torch()
        with self._ws_lock:
            if self._dir is not None:
                return self._dir or None
            L = _native.lib()
            d = _native.RlfcDir()
            if L.rlfc_dir_plan(self.ref, ctypes.byref(d)) != _native.RLFC_OK:
                self._dir = False
                return None
            t0 = time.perf_counter()
            dev = self.device
            with torch.cuda.device(dev):
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                scratch = torch.empty(d.scratch_bytes, dtype=torch.uint8,
                                      device=dev)
                blob_off = torch.empty(d.n_blobs + 1, dtype=torch.int32,
                                       device=dev)
                flagged = torch.empty(max(1, d.nrec), dtype=torch.int32,
                                      device=dev)
                root_rgb = torch.empty(max(16, d.root_rgb_bytes),
                                       dtype=torch.uint8, device=dev)
                tables = torch.empty(_native.DIR_TABLE_BYTES,
                                     dtype=torch.uint8, device=dev)
                d.tables = tables.data_ptr()
                d.scratch = scratch.data_ptr()
                d.blob_off = blob_off.data_ptr()
                d.flagged = flagged.data_ptr()
                d.root_rgb = root_rgb.data_ptr()
                rc = L.rlfc_dir_size(self.ref, ctypes.byref(d), _stream())
                if rc == _native.RLFC_ERR_ARGUMENT:
                    self._dir = False
                    return None
                _native.check(rc, "rlfc_dir_size")
                blobs = torch.empty(d.blob_bytes + 64, dtype=torch.uint8,
                                    device=dev)
                d.blobs = blobs.data_ptr()
                _native.check(L.rlfc_dir_build(self.ref, ctypes.byref(d),
                                               _stream()), "rlfc_dir_build")
                torch.cuda.synchronize(dev)
                build_ms = (time.perf_counter() - t0) * 1e3
            d.scratch = None
            del scratch
            self._dir = Directory(d, blobs, blob_off, flagged, root_rgb,
                                  tables, build_ms)
            return self._dir

    def index_view(self):
        """The prepared record index as an rlfc_index_view (B = 4), from any
        staged workspace of this field (its index part is read-only after
        prepare; the view keeps that workspace alive), or None."""
        v = self._index_view
        if v is not None:
            return v or None
        torch = _torch()
        with self._ws_lock:
            have = next(iter(self._ws.values()), None)
        ws = None
        if have is not None:
            ws = (have[0], self._ws_bytes, self._present)
        else:
            with torch.cuda.device(self.device):
                cur = torch.cuda.current_stream(self.device)
                got = self.staged_workspace(cur.cuda_stream)
                if got is not None:
                    ws = got[:3]
                    cur.synchronize()
        view = False
        if ws is not None:
            iv = _native.IndexView()
            if _native.lib().rlfc_staged_index_view(self.ref, ws[0].data_ptr(), ws[1], ws[2],
                                                    ctypes.byref(iv)) == _native.RLFC_OK:
                iv._ws_ref = ws[0]
                view = iv
        self._index_view = view
        return view or None

    def staged_workspace(self, stream_handle):
        """(tensor, bytes, present_total, n_flagged) for the staged decode on one CUDA
        stream, allocated and prepared on first use.  present_total (the
        number of present nodes over all records) is counted on the device
        once per field; rlfc_staged_prepare then builds the stream-invariant
        record index (payload entries, record tables) and the root colours
        into the workspace, which also holds the decoded residuals of each
        step (rlfc_staged.cu)."""
        torch = _torch()
        L = _native.lib()
        with self._ws_lock:
            if self._present is None:
                cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
                with torch.cuda.device(self.device):
                    _native.check(L.rlfc_count_present(self.ref, cnt.data_ptr(),
                                                       _stream()),
                                  "rlfc_count_present")
                self._present = int(cnt.item())
                need = ctypes.c_uint64(0)
                rc = L.rlfc_decode_workspace_bytes(self.ref, self._present,
                                                   ctypes.byref(need))
                self._ws_bytes = int(need.value) if rc == _native.RLFC_OK \
                    else 0
            if not self._ws_bytes:
                return None
            ws = self._ws.get(stream_handle)
            if ws is None:
                ws = torch.empty(self._ws_bytes, dtype=torch.uint8,
                                 device=self.device)
                # the record index (payload entries, record tables), the
                # anomaly list and the root colours are stream-invariant:
                # built once per workspace
                nflag = ctypes.c_int32(0)
                with torch.cuda.device(self.device):
                    _native.check(L.rlfc_staged_prepare(
                        self.ref, ws.data_ptr(), self._ws_bytes,
                        self._present, ctypes.byref(nflag), stream_handle),
                        "rlfc_staged_prepare")
                ws = (ws, int(nflag.value))
                self._ws[stream_handle] = ws
            return ws[0], self._ws_bytes, self._present, ws[1]

    @property
    def hbm_bytes(self):
        return sum(t.numel() * t.element_size()
                   for t in self.srv + self.offsets + [self.roots])


class Directory:
    """Device record directory of one DeviceField (rlfc_dir_build)."""

    def __init__(self, c, blobs, blob_off, flagged, root_rgb, tables,
                 build_ms):
        self.c = c
        self.ref = ctypes.byref(c)
        self.blobs, self.blob_off = blobs, blob_off
        self.flagged, self.root_rgb, self.tables = flagged, root_rgb, tables
        self.build_ms = build_ms

    @property
    def n_flagged(self):
        return int(self.c.n_flagged)

    @property
    def blob_bytes(self):
        return int(self.c.blob_bytes)

    @property
    def hbm_bytes(self):
        return sum(t.numel() * t.element_size() for t in
                   (self.blobs, self.blob_off, self.flagged, self.root_rgb,
                    self.tables))


def tile_bytes_max(header, offsets):
    """Staging need of the fused decode's tiles: the largest compressed size
    of max(1, 32/B) consecutive records of one block row, summed over the
    channels, plus alignment slack per channel (rlfc_b200.h)."""
    wb, hb = header.block_grid
    nb = 1 if header.block_size >= 16 else 32 // header.block_size
    total = np.zeros((hb, -(-wb // nb)), dtype=np.int64)
    for c in range(3):
        offs = np.asarray(offsets[c], dtype=np.int64)
        ends = np.append(offs[1:], header.section_lengths[c][2])
        sizes = (ends - offs).reshape(hb, wb)
        pad = (-wb) % nb
        sizes = np.pad(sizes, ((0, 0), (0, pad)))
        total += sizes.reshape(hb, -1, nb).sum(axis=2) + 32
    return int(min(total.max(), 2**31 - 1)) if total.size else 0


@dataclass(frozen=True)
class DecoderState:
    """Immutable, request-ready state (reference decoder.py:20-28) plus the
    per-GPU device copies."""
    header: container.RlfcHeader
    data: bytes
    _root_host: object           # (rsx, rsy, 3, Hp, Wp) int32, unbiased, or None (on the GPU)
    offsets: tuple               # per channel u64 array, one per block
    srv: tuple                   # per channel uint8 view of the SRV stream
    chains: np.ndarray           # (S, T, h) ascending serial ancestor indices
    m_nodes: int
    _devices: dict = field(default_factory=dict, compare=False, repr=False)
    _roots_dev: dict = field(default_factory=dict, compare=False, repr=False)
    _lock: object = field(default_factory=threading.Lock, compare=False,
                          repr=False)

    @property
    def root_planes(self) -> np.ndarray:
        """(rsx, rsy, 3, Hp, Wp) int32 root planes, bias removed (reference
        DecoderState.root_planes).  When the roots were decoded on the GPU at
        init, the host copy is made on first use."""
        if self._root_host is None:
            t = next(iter(self._roots_dev.values()))
            object.__setattr__(self, "_root_host", t.cpu().numpy().astype(np.int32))
        return self._root_host

    def device_field(self, device=None) -> DeviceField:
        """The stream's HBM copy on `device` (default: current CUDA device),
        uploaded on first use."""
        torch = _torch()
        _native.lib()
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if device is None else torch.device(device)
        key = dev.index
        with self._lock:
            df = self._devices.get(key)
            if df is None:
                rd = self._roots_dev.get(key)
                df = DeviceField(self.header, self.srv, self.offsets,
                                 None if rd is not None else self.root_planes,
                                 dev, roots_dev=rd)
                self._devices[key] = df
        return df


def init(stream: bytes, device=None) -> DecoderState:
    """Parse a stream and upload it to the GPU (reference decoder.py:31-48)."""
    header = container.parse_header(stream)
    container.check_stream_length(header, stream)
    data = bytes(stream)
    torch = _torch()
    _native.lib()                       # no CUDA device: NativeUnavailable
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if device is None else torch.device(device)
    # PNG roots: inflated on host threads, unfiltered on the GPU; anything
    # unusual goes through Pillow (the reference's decoder and errors)
    got = container.parse_roots_device(data, header, dev)
    roots_dev, roots = got, None
    if got is None:
        roots = container.parse_roots(data, header)
    offsets = tuple(container.parse_offsets(data, header, c) for c in range(3))
    srv = tuple(container.srv_section(data, header, c) for c in range(3))
    chains = container.all_chains(header.s_count, header.t_count,
                                  header.tree_height)
    m = container.total_srv_nodes(header.s_count, header.t_count,
                                  header.tree_height)
    state = DecoderState(header=header, data=data, _root_host=roots,
                         offsets=offsets, srv=srv, chains=chains, m_nodes=m)
    if roots_dev is not None:
        state._roots_dev[dev.index] = roots_dev
    state.device_field(dev)
    return state


# --- argument checks and error mapping (decoder.py:51-70) ---------------------

def _check_indices(state, s, t, bx=0, by=0):
    hdr = state.header
    if not (0 <= s < hdr.s_count and 0 <= t < hdr.t_count):
        raise IndexError(f"image index ({s}, {t}) outside grid")
    wb, hb = hdr.block_grid
    if not (0 <= bx < wb and 0 <= by < hb):
        raise IndexError(f"block index ({bx}, {by}) outside block grid")


def _check_level(state, stop_level):
    if not 0 <= stop_level <= state.header.tree_height:
        raise ValueError(f"stop level {stop_level} outside [0, "
                         f"{state.header.tree_height}]")


def _check_requests(state, req, ncol):
    """Range checks of batched requests (decoder.py:51-63 per request): s, t,
    block indices inside the grid, channel in [-3, 3) (Python indexing, as
    the reference's root_planes[..., c] / srv[c]) and, for blocks, the stop
    level in [0, h].  Raises IndexError / ValueError like the reference;
    returns the requests with negative channels normalised."""
    hdr = state.header
    wb, hb = hdr.block_grid
    S, T, h = hdr.s_count, hdr.t_count, hdr.tree_height
    torch = _torch()
    if isinstance(req, torch.Tensor):
        if req.numel() == 0:
            return req
        lo = req.min(dim=0).values.cpu().numpy()
        hi = req.max(dim=0).values.cpu().numpy()
    else:
        if req.size == 0:
            return req
        lo, hi = req.min(axis=0), req.max(axis=0)
    if lo[0] < 0 or hi[0] >= S or lo[1] < 0 or hi[1] >= T:
        raise IndexError("image index outside grid")
    if ncol == 6:
        if lo[2] < 0 or hi[2] >= wb or lo[3] < 0 or hi[3] >= hb:
            raise IndexError("block index outside block grid")
        c, k = 4, 5
        if lo[k] < 0 or hi[k] > h:
            raise ValueError(f"stop level outside [0, {h}]")
    else:
        c = 2
    if lo[c] < -3 or hi[c] >= 3:
        raise IndexError("index out of bounds for axis 2 with size 3")
    if lo[c] < 0:
        req = req.clone() if isinstance(req, torch.Tensor) else req.copy()
        req[:, c] %= 3
    return req


def _raise_status(code):
    if code == 1:
        raise FormatError("corrupt coded pack in SRV payload")
    if code == 2:
        raise FormatError("descriptor outside range table")


def _raise_word(word):
    got = _native.decode_status_word(word)
    if got is not None:
        _raise_status(got[1])


def _stream():
    return _torch().cuda.current_stream().cuda_stream


# --- batched device API ------------------------------------------------------

def decode_blocks(state, requests, device=None, raise_errors=True):
    """Decode a batch of blocks on the GPU.

    requests: (n, 6) ints (s, t, bx, by, channel, stop_level).  Returns
    (CUDA int32 tensor (n, B, B), CUDA int32 status tensor (n,)).  Host
    requests are range-checked first (IndexError / ValueError as
    decoder.py:51-63); device requests are checked by the kernel (status 3).
    With raise_errors the first failing request (lowest index) raises the
    reference's error.
    """
    torch = _torch()
    df = state.device_field(device)
    if isinstance(requests, torch.Tensor) and requests.is_cuda:
        # device-resident requests are range-checked by the kernel (code 3)
        req = requests.to(torch.int32).reshape(-1, 6).contiguous()
    else:
        req = _check_requests(state, np.ascontiguousarray(
            requests, dtype=np.int32).reshape(-1, 6), 6)
        req = torch.as_tensor(req).to(df.device, non_blocking=True)
    n = req.shape[0]
    b = state.header.block_size
    out = torch.empty((n, b, b), dtype=torch.int32, device=df.device)
    status = torch.zeros(n, dtype=torch.int32, device=df.device)
    with torch.cuda.device(df.device):
        stream = _stream()
        # the prepared index pays from ~4k requests on; smaller batches use
        # it too once the field has one (its index part is read-only)
        if n >= 4096:
            ws = df.staged_workspace(stream)
        else:
            with df._ws_lock:
                have = next(iter(df._ws.values()), None)
            ws = None if have is None else (have[0], df._ws_bytes, df._present)
        rc = _native.RLFC_ERR_ARGUMENT
        if ws is not None:
            # large batches: the prepared record index (no record walks)
            rc = _native.lib().rlfc_decode_blocks_indexed(
                df.ref, ws[0].data_ptr(), ws[1], ws[2], req.data_ptr(), n,
                out.data_ptr(), status.data_ptr(), stream)
        if rc == _native.RLFC_ERR_ARGUMENT:
            rc = _native.lib().rlfc_decode_blocks(
                df.ref, req.data_ptr(), n, out.data_ptr(), status.data_ptr(),
                stream)
        _native.check(rc, "rlfc_decode_blocks")
    if raise_errors and n:
        st = status.cpu().numpy()
        bad = np.flatnonzero(st)
        if bad.size:
            if st[bad[0]] == 3:
                _check_requests(state, req.cpu().numpy(), 6)     # raises
                raise IndexError("block request out of range")
            _raise_status(int(st[bad[0]]))
    return out, status


def decode_planes(state, planes, stop_level=0, device=None):
    """(n, Hp, Wp) int32 CUDA tensor of padded planes for (s, t, c) triples."""
    torch = _torch()
    df = state.device_field(device)
    _check_level(state, stop_level)
    req = _check_requests(state, np.ascontiguousarray(
        planes, dtype=np.int32).reshape(-1, 3), 3)
    req = torch.as_tensor(req).to(df.device)
    n = req.shape[0]
    wp, hp = state.header.padded_dims
    out = torch.empty((n, hp, wp), dtype=torch.int32, device=df.device)
    status = torch.zeros(1, dtype=torch.int64, device=df.device)
    with torch.cuda.device(df.device):
        _native.check(_native.lib().rlfc_decode_planes(
            df.ref, stop_level, req.data_ptr(), n, out.data_ptr(),
            status.data_ptr(), _stream()), "rlfc_decode_planes")
    _raise_word(status.cpu().item())
    return out


KERNELS = ("auto", "dir", "staged", "fused", "simple")


def decode_field(state, stop_level=0, images=None, rows=None, out=None,
                 device=None, kernel="auto", check=True):
    """Decode many camera images straight into an RGB8 CUDA tensor.

    images: None for the whole (S, T) grid -- the result is (S, T, H, W, 3)
    -- or a sequence of (s, t) pairs -- the result is (n, H, W, 3) in that
    order.  rows: optional block-row band (by_lo, by_hi); the result then
    holds only pixel rows [by_lo*B, min(by_hi*B, H)).  kernel: "auto" (=
    "staged"), "staged" (payload decode -> blend over the prepared record
    index, rlfc_staged.cu; falls back to "fused" outside its envelope),
    "dir" (one kernel over the tile-major device record directory,
    rlfc_dir.cu; slower at cfg2, kept as an alternative and cross-check),
    "fused" (the single tiled kernel, rlfc_field.cu) or "simple" (per-block
    kernel).  With check, a
    corrupt stream raises the FormatError the reference raises first.
    Returns (tensor, status) where status is the device status word tensor.
    """
    torch = _torch()
    hdr = state.header
    _check_level(state, stop_level)
    df = state.device_field(device)
    S, T, W, H, B = hdr.s_count, hdr.t_count, hdr.width, hdr.height, \
        hdr.block_size
    _, hb = hdr.block_grid
    by_lo, by_hi = (0, hb) if rows is None else (int(rows[0]), int(rows[1]))
    if not 0 <= by_lo <= by_hi <= hb:
        raise ValueError(f"block-row band {rows} outside [0, {hb}]")
    nrows = max(0, min(by_hi * B, H) - by_lo * B)
    slots_t = trows_t = None
    if images is None:
        shape = (S, T, nrows, W, 3)
        nimg = S * T
    else:
        pairs = [tuple(map(int, p)) for p in images]
        slots = np.full(S * T, -1, dtype=np.int32)
        for i, (s, t) in enumerate(pairs):
            _check_indices(state, s, t)
            if slots[s * T + t] >= 0:
                raise ValueError(f"image ({s}, {t}) requested twice")
            slots[s * T + t] = i
        shape = (len(pairs), nrows, W, 3)
        nimg = len(pairs)
        slots_t = torch.from_numpy(slots).to(df.device)
        trows_t = torch.tensor(sorted({t for _, t in pairs}), dtype=torch.int32,
                               device=df.device)
    if out is None:
        out = torch.empty(shape, dtype=torch.uint8, device=df.device)
    elif tuple(out.shape) != shape or out.dtype != torch.uint8 or \
            not out.is_contiguous():
        raise ValueError(f"out must be a contiguous uint8 tensor {shape}")
    status = torch.zeros(1, dtype=torch.int64, device=df.device)
    if kernel not in KERNELS:
        raise ValueError(f"unknown decode kernel {kernel!r}")
    if nimg and nrows:
        L = _native.lib()
        slots_p = None if slots_t is None else slots_t.data_ptr()
        with torch.cuda.device(df.device):
            done = False
            if kernel == "dir" and slots_t is None:
                dr = df.directory()
                if dr is not None:
                    rc = L.rlfc_decode_field_dir(
                        df.ref, dr.ref, stop_level, by_lo, by_hi,
                        out.data_ptr(), nrows * W * 3, W * 3,
                        status.data_ptr(), _stream())
                    if rc != _native.RLFC_ERR_ARGUMENT:
                        _native.check(rc, "rlfc_decode_field_dir")
                        done = True
            if not done and kernel in ("auto", "dir", "staged"):
                stream = _stream()
                ws = df.staged_workspace(stream)
                if ws is not None:
                    with df.enqueue_lock:
                        rc = L.rlfc_decode_field_staged(
                            df.ref, stop_level, slots_p, by_lo, by_hi,
                            out.data_ptr(), nrows * W * 3, W * 3,
                            ws[0].data_ptr(), ws[1], ws[2], ws[3],
                            None if trows_t is None else trows_t.data_ptr(),
                            0 if trows_t is None else trows_t.numel(),
                            status.data_ptr(), stream)
                    if rc != _native.RLFC_ERR_ARGUMENT:
                        _native.check(rc, "rlfc_decode_field_staged")
                        done = True
            if not done:
                fn = L.rlfc_decode_field_simple if kernel == "simple" else \
                    L.rlfc_decode_field
                _native.check(fn(
                    df.ref, stop_level, slots_p, by_lo, by_hi,
                    out.data_ptr(), nrows * W * 3, W * 3, status.data_ptr(),
                    _stream()), "rlfc_decode_field")
    if check:
        _raise_word(status.cpu().item())
    return out, status


def decode_field_slots(state, stop_level, slots, n, device=None, rows=None):
    """decode_field for a prebuilt device slot table (slots[s*T + t] = output
    index or -1, n outputs): the renderer's tap-camera decode.  rows: the
    camera rows holding requested views (host ints; None = all rows).
    Returns (field (n, H, W, 3), status word tensor) without
    synchronising."""
    torch = _torch()
    hdr = state.header
    df = state.device_field(device)
    trows = None if rows is None else torch.tensor(sorted(set(int(r) for r in rows)),
                                                   dtype=torch.int32, device=df.device)
    W, H = hdr.width, hdr.height
    out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=df.device)
    status = torch.zeros(1, dtype=torch.int64, device=df.device)
    L = _native.lib()
    hb = hdr.block_grid[1]
    with torch.cuda.device(df.device):
        stream = _stream()
        ws = df.staged_workspace(stream)
        rc = _native.RLFC_ERR_ARGUMENT
        if ws is not None:
            with df.enqueue_lock:
                rc = L.rlfc_decode_field_staged(
                    df.ref, stop_level, slots.data_ptr(), 0, hb,
                    out.data_ptr(), H * W * 3, W * 3, ws[0].data_ptr(), ws[1],
                    ws[2], ws[3], None if trows is None else trows.data_ptr(),
                    0 if trows is None else trows.numel(), status.data_ptr(),
                    stream)
        if rc == _native.RLFC_ERR_ARGUMENT:
            rc = L.rlfc_decode_field(df.ref, stop_level, slots.data_ptr(), 0,
                                     hb, out.data_ptr(), H * W * 3, W * 3,
                                     status.data_ptr(), stream)
        _native.check(rc, "rlfc_decode_field")
    return out, status


def bise_decode_batch(payloads, descs, count, device=None):
    """Decode many BISE payloads on the GPU (kernels.bise_decode_core).

    Returns (values uint32 (n, count) numpy, status int32 (n,) numpy).
    """
    torch = _torch()
    _native.lib()
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if device is None else torch.device(device)
    blobs = [bytes(p) for p in payloads]
    offs = np.zeros(len(blobs), dtype=np.int64)
    pos = 0
    for i, b in enumerate(blobs):
        offs[i] = pos
        pos += len(b)
    data = np.zeros(pos + SRV_TAIL_PAD, dtype=np.uint8)
    data[:pos] = np.frombuffer(b"".join(blobs), dtype=np.uint8)
    d_data = torch.from_numpy(data).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    d_desc = torch.from_numpy(np.asarray(descs, dtype=np.uint8)).to(dev)
    n = len(blobs)
    out = torch.zeros((n, count), dtype=torch.int32, device=dev)
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _native.check(_native.lib().rlfc_bise_decode(
            d_data.data_ptr(), d_offs.data_ptr(), d_desc.data_ptr(), n, count,
            out.data_ptr(), status.data_ptr(), _stream()), "rlfc_bise_decode")
    return out.cpu().numpy().view(np.uint32), status.cpu().numpy()


# --- reference-signature API ---------------------------------------------------

MAILBOX_BYTES = 64 + 16 * 88                  # rlfc_mailbox (include/rlfc_b200.h)
_REQ = struct.Struct("<6i")                    # rlfc_block_call.req
_REQ_OFF = 48
BLOCK_SERVER_IDLE_NS = 1_000_000              # resident server exits after 1 ms idle


def _stop_server(fn, mailbox, stream):
    fn(mailbox.data_ptr(), stream.cuda_stream)


class _BlockScratch:
    """Per-thread state for single-block requests: a mailbox in pinned host
    memory and a private CUDA stream.  A request is one ctypes call into
    rlfc_block_server_request: a resident one-warp server kernel on that
    stream (started on demand, gone after 1 ms without requests) reads the
    request from the mailbox over PCIe and writes the block back, so a
    request in a stream of requests costs no kernel launch."""

    def __init__(self, df, b):
        torch = _torch()
        self.b = b
        self.mailbox = torch.zeros(MAILBOX_BYTES, dtype=torch.uint8).pin_memory()
        self.out_np = np.zeros(b * b + 1, dtype=np.int32)
        self.out_block = self.out_np[:b * b].reshape(b, b)
        self.stream = torch.cuda.Stream(device=df.device)
        L = _native.lib()
        self.args = (df.ref, self.mailbox.data_ptr(), self.stream.cuda_stream)
        self.out_ptr = self.out_np.ctypes.data
        # the prepared record index of the field (any workspace: its index
        # part is read-only after prepare): B = 4 requests skip the record
        # walk (one lane per chain level)
        self.index = df.index_view() if b == 4 else None
        self.index_ptr = ctypes.addressof(self.index) if self.index is not None else None
        # the whole call in one struct: per request only req changes
        self.call = _native.BlockCall(ctypes.addressof(df.cfield), self.mailbox.data_ptr(), self.index_ptr,
                                      self.stream.cuda_stream, BLOCK_SERVER_IDLE_NS, self.out_ptr)
        self.call_ptr = ctypes.addressof(self.call)
        hdr = df.header
        self.dims = (hdr.s_count, hdr.t_count) + tuple(hdr.block_grid) + (hdr.tree_height,)
        self.bsq = b * b
        self.call_fn = L.rlfc_block_server_call
        self.fn = L.rlfc_block_server_request
        # the server must be gone before the mailbox (or the field) is reused
        weakref.finalize(self, _stop_server, L.rlfc_block_server_stop,
                         self.mailbox, self.stream)


def _block_scratch(state):
    """The calling thread's single-block scratch for this state's field on
    the current device.  It lives on the DeviceField (keyed by thread), so it
    is released with the state; nothing module-level holds the state."""
    df = _field_on(state)
    key = threading.get_ident()
    sc = df.block_scratch.get(key)
    if sc is None:
        sc = df.block_scratch[key] = _BlockScratch(df, state.header.block_size)
    return sc


def decode_block_progressive(state: DecoderState, image_index, block_index,
                             channel, stop_level):
    """One B x B block summing SRV levels >= stop_level (decoder.py:81-106)."""
    s, t = image_index
    bx, by = block_index
    sc = _block_scratch(state)
    S, T, wb, hb, h = sc.dims
    if not (0 <= s < S and 0 <= t < T):
        _check_indices(state, s, t, bx, by)
    if not (0 <= bx < wb and 0 <= by < hb):
        _check_indices(state, s, t, bx, by)
    if not 0 <= stop_level <= h:
        _check_level(state, stop_level)
    # the reference indexes root_planes[..., channel] and srv[channel]
    # (decoder.py:73-78, 99-101): Python indexing, so -3..-1 alias 0..2
    if not -3 <= channel < 3:
        raise IndexError(f"index {channel} is out of bounds for axis 2 with "
                         "size 3")
    _REQ.pack_into(sc.call, _REQ_OFF, s, t, bx, by, int(channel) % 3, stop_level)
    rc = sc.call_fn(sc.call_ptr)
    if rc:
        _native.check(rc, "rlfc_block_server_request")
    code = sc.out_np.item(sc.bsq)
    if code:
        _raise_status(code)
    return sc.out_block.copy()


def decode_block(state: DecoderState, image_index, block_index, channel):
    """Fully decode one block of one channel plane (decoder.py:109-112)."""
    return decode_block_progressive(state, image_index, block_index, channel, 0)


def decode_block_traced(state: DecoderState, image_index, block_index,
                        channel, stop_level=0):
    """decode_block plus the absolute SRV byte ranges a decode reads.

    Host-side read-locality mirror (decoder.py:115-162): the ranges come from
    a walk of the record on the host; the block itself is decoded on the GPU.
    """
    s, t = image_index
    bx, by = block_index
    _check_indices(state, s, t, bx, by)
    _check_level(state, stop_level)
    hdr = state.header
    wb, _ = hdr.block_grid
    starts, _ = container.section_offsets(hdr)
    rec = starts[channel][2] + int(state.offsets[channel][by * wb + bx])
    nbm = (state.m_nodes + 7) >> 3
    ranges = [(rec, rec + nbm)]
    bits = np.unpackbits(np.frombuffer(state.data[rec:rec + nbm], np.uint8),
                         bitorder="little")
    targets = set(int(v) for v in
                  state.chains[s, t, :hdr.tree_height - stop_level])
    top = max(targets) if targets else -1
    pbytes = payload_bytes_table(hdr.block_size ** 2)
    cursor = rec + nbm
    for node in np.flatnonzero(bits[:top + 1]):
        desc = state.data[cursor]
        ranges.append((cursor, cursor + 1))
        if desc >= len(RANGE_TABLE):
            raise FormatError(f"descriptor {desc} outside range table")
        if int(node) in targets:
            ranges.append((cursor + 1, cursor + 1 + int(pbytes[desc])))
        cursor += 1 + int(pbytes[desc])
    block = decode_block_progressive(state, image_index, block_index, channel,
                                     stop_level)
    return block, ranges


def _to_host(t):
    """Device tensor -> numpy through pinned memory (torch's caching host
    allocator): the copy runs at PCIe speed instead of through the driver's
    pageable staging, and the returned array owns the pinned block."""
    torch = _torch()
    if t.numel() * t.element_size() > (256 << 20):
        return _to_host_big(t)                 # big results: no pinned-cache growth
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


_BOUNCE = 64 << 20
# one process-wide ring of pinned bounce buffers and copy pool: large
# results are PCIe-bound, so concurrent callers take turns (_bounce_lock)
# instead of each pinning its own 192 MB
_bounce = {}
_bounce_lock = threading.Lock()


def _to_host_big(t):
    """Large device tensor -> fresh (pageable) numpy array: chunks go through
    a ring of three pinned bounce buffers at PCIe speed while host threads
    copy the previous chunk into place (page faults of the fresh array spread
    over the threads).  A plain pageable .cpu() of cfg2's 909 MB field took
    426 ms."""
    from concurrent.futures import ThreadPoolExecutor
    torch = _torch()
    src = t.contiguous().view(torch.uint8).reshape(-1)
    n = src.numel()
    out = np.empty(n, dtype=np.uint8)
    with _bounce_lock:
        if not _bounce:
            _bounce["ring"] = [torch.empty(_BOUNCE, dtype=torch.uint8).pin_memory() for _ in range(3)]
            _bounce["pool"] = ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
        return _to_host_ring(t, src, n, out, _bounce["ring"], _bounce["pool"])


def _to_host_ring(t, src, n, out, ring, pool):
    """_to_host_big's pipeline over the shared ring (caller holds _bounce_lock)."""
    torch = _torch()
    stream = torch.cuda.Stream(device=t.device)
    stream.wait_stream(torch.cuda.current_stream(t.device))
    chunks = [(a, min(n, a + _BOUNCE)) for a in range(0, n, _BOUNCE)]
    events = []
    pending = []

    def issue(i):
        a, b = chunks[i]
        with torch.cuda.stream(stream):
            ring[i % 3][:b - a].copy_(src[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        events.append(ev)

    def drain(i):
        a, b = chunks[i]
        events[i].synchronize()
        buf = ring[i % 3].numpy()
        parts = 8
        step = -(-(b - a) // parts)
        futs = [pool.submit(np.copyto, out[a + j:min(b, a + j + step)], buf[j:min(b - a, j + step)])
                for j in range(0, b - a, step)]
        return futs

    for i in range(min(2, len(chunks))):
        issue(i)
    for i in range(len(chunks)):
        futs = drain(i)
        for f in pending:
            f.result()
        pending = futs
        if i + 2 < len(chunks):
            # ring slot (i + 2) % 3 was drained two steps ago (its copies done)
            issue(i + 2)
    for f in pending:
        f.result()
    return out.view(np.dtype(str(t.dtype).replace("torch.", ""))).reshape(tuple(t.shape))


def decode_plane(state: DecoderState, s, t, channel, stop_level=0):
    """One image channel plane at padded dims, int32 (decoder.py:165-184)."""
    _check_indices(state, s, t)
    _check_level(state, stop_level)
    # root_planes[..., channel] / srv[channel] in the reference: Python
    # indexing, so -3..-1 alias 0..2 and anything else is an IndexError
    if not -3 <= channel < 3:
        raise IndexError(f"index {channel} is out of bounds for axis 2 with "
                         "size 3")
    channel = int(channel) % 3
    if stop_level == state.header.tree_height:
        h = state.header.tree_height
        return state.root_planes[s >> h, t >> h, channel].copy()
    # one native call: request staged, k_decode_planes, pinned result
    torch = _torch()
    hdr = state.header
    # the current device's field (device_field() default): no device switch
    df = _field_on(state)
    wp, hp = hdr.padded_dims
    host_stage, dev_stage, word = _image_buffers(df, 64)
    plane = torch.empty((hp, wp), dtype=torch.int32, device=df.device)
    res = torch.empty((hp, wp), dtype=torch.int32, pin_memory=True)
    iv = df.index_view() if hdr.block_size == 4 else None
    rc = _native.lib().rlfc_decode_plane_host(
        df.ref, stop_level, int(s), int(t), channel, plane.data_ptr(), res.data_ptr(),
        host_stage.data_ptr(), dev_stage.data_ptr(), word.ctypes.data,
        None if iv is None else ctypes.byref(iv),
        torch._C._cuda_getCurrentRawStream(df.device.index))
    _native.check(rc, "rlfc_decode_plane_host")
    _raise_word(int(word[0]))
    return res.numpy()


_img_tls = threading.local()


def _image_buffers(df, need):
    """Per-thread, per-device staging of the one-call image / plane decodes:
    (pinned host buffer, device buffer, status word), grown on demand."""
    torch = _torch()
    key = df.device.index
    bufs = getattr(_img_tls, "bufs", None)
    if bufs is None:
        bufs = _img_tls.bufs = {}
    b = bufs.get(key)
    if b is None or b[0].numel() < need:
        cap = max(4096, 1 << (need - 1).bit_length())
        b = bufs[key] = (torch.empty(cap, dtype=torch.uint8).pin_memory(),
                         torch.empty(cap, dtype=torch.uint8, device=df.device),
                         np.zeros(1, dtype=np.uint64))
    return b


def decode_image(state: DecoderState, image_index, stop_level=0):
    """One camera image as true-dims RGB8 (decoder.py:187-194): one native
    call (rlfc_decode_image_host) stages the slot table, decodes and brings
    the image back into a pinned array the result owns."""
    torch = _torch()
    s, t = image_index
    _check_indices(state, s, t)
    _check_level(state, stop_level)
    hdr = state.header
    # the current device's field (device_field() default): no device switch
    df = _field_on(state)
    L = _native.lib()
    host_stage, dev_stage, word = _image_buffers(df, 48 + 4 * hdr.s_count * hdr.t_count + 4 * 65)
    img = torch.empty((hdr.height, hdr.width, 3), dtype=torch.uint8, device=df.device)
    res = torch.empty((hdr.height, hdr.width, 3), dtype=torch.uint8, pin_memory=True)
    stream = torch._C._cuda_getCurrentRawStream(df.device.index)
    ws = df.staged_workspace(stream)
    args = (None, 0, 0, 0) if ws is None else (ws[0].data_ptr(), ws[1], ws[2], ws[3])
    with df.enqueue_lock:
        rc = L.rlfc_decode_image_host(df.ref, stop_level, *args, int(s), int(t), img.data_ptr(),
                                      res.data_ptr(), host_stage.data_ptr(), dev_stage.data_ptr(),
                                      host_stage.numel(), word.ctypes.data, stream)
    _native.check(rc, "rlfc_decode_image_host")
    _raise_word(int(word[0]))
    return res.numpy()


def decode_all(state: DecoderState, stop_level=0) -> LightFieldGrid:
    """The whole grid as a LightFieldGrid (decoder.py:197-210)."""
    hdr = state.header
    out, _ = decode_field(state, stop_level)
    return LightFieldGrid(hdr.s_count, hdr.t_count, hdr.width, hdr.height,
                          _to_host(out),
                          grid_positions(hdr.s_count, hdr.t_count),
                          default_geometry(hdr.s_count, hdr.t_count))


def planes_to_rgb(planes):
    """Host helper: three int32 planes -> clamped RGB8 (colorspace.py:46-56)."""
    return colorspace.planes_to_grid(planes)


class HostPipeline:
    """End-to-end decode with host buffers, the path a host application
    takes: every run() uploads the compressed sections (SRV + offsets) and
    the root planes from pinned host memory, runs the staged decode, and
    copies the RGB8 result into pinned host memory.  The rows are split into
    `bands` block-row bands pipelined over three CUDA streams (upload of band
    i+1 | decode of band i | download of band i-1), so the PCIe transfers in
    both directions overlap each other and the decode.  h2d_bytes / d2h_bytes
    are the bytes those copies move per run."""

    def __init__(self, state, rows=None, device=None, bands=8):
        torch = _torch()
        self.state = state
        hdr = state.header
        hb = hdr.block_grid[1]
        self.rows = (0, hb) if rows is None else tuple(rows)
        B = hdr.block_size
        self.rows_px = max(0, min(self.rows[1] * B, hdr.height) -
                           self.rows[0] * B)
        src = state.device_field(device)
        self.df = DeviceField(hdr, state.srv, state.offsets,
                              state.root_planes, src.device)
        self.host_srv = [t.cpu().pin_memory() for t in self.df.srv]
        self.host_off = [t.cpu().pin_memory() for t in self.df.offsets]
        self.host_roots = self.df.roots.cpu().pin_memory()
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in
                             self.host_srv + self.host_off) + \
            self.host_roots.numel() * self.host_roots.element_size()
        shape = (hdr.s_count, hdr.t_count, self.rows_px, hdr.width, 3)
        self.out = torch.empty(shape, dtype=torch.uint8, device=src.device)
        self.out_host = torch.empty(shape, dtype=torch.uint8).pin_memory()
        self.d2h_bytes = self.out_host.numel()
        self.status = torch.zeros(1, dtype=torch.int64, device=src.device)
        lo, hi = self.rows
        # banded uploads need the records in block order (a corrupt stream
        # may not have them): else one band with everything uploaded
        self.monotone = all(bool(np.all(np.diff(o.astype(np.int64)) >= 0))
                            for o in state.offsets)
        n = max(1, min(bands, hi - lo)) if self.monotone else 1
        cuts = [lo + (hi - lo) * i // n for i in range(n + 1)]
        self.bands = [(a, b) for a, b in zip(cuts, cuts[1:]) if b > a]
        self.streams = [torch.cuda.Stream(device=src.device) for _ in range(3)]

    def _srv_range(self, c, lo, hi):
        hdr = self.state.header
        wb, hb = hdr.block_grid
        if not self.monotone:
            return 0, self.host_srv[c].numel()
        offs = self.state.offsets[c]
        a = int(offs[lo * wb]) if lo < hb else len(self.state.srv[c])
        b = int(offs[hi * wb]) if hi < hb else len(self.state.srv[c])
        if hi >= hb:
            b = self.host_srv[c].numel()              # + the zero tail padding
        return a, b

    def run(self):
        torch = _torch()
        hdr = self.state.header
        L = _native.lib()
        W, B = hdr.width, hdr.block_size
        s_in, s_dec, s_out = self.streams
        df = self.df
        rt = df.roots
        esz = rt.element_size()
        plane = hdr.padded_dims[0] * hdr.padded_dims[1] * esz
        row_b = hdr.padded_dims[0] * B * esz             # one block row of a root plane
        nplanes = rt.numel() * esz // plane if plane else 0
        img = self.rows_px * W * 3
        self.status.zero_()
        cur = torch.cuda.current_stream(df.device)
        for s in self.streams:
            s.wait_stream(cur)
        with torch.cuda.device(df.device):
            ws = df.staged_workspace(s_dec.cuda_stream)
            with torch.cuda.stream(s_in):
                for d, h in zip(df.offsets, self.host_off):
                    d.copy_(h, non_blocking=True)
            for lo, hi in self.bands:
                with torch.cuda.stream(s_in):
                    for c in range(3):
                        a, b = self._srv_range(c, lo, hi)
                        if b > a:
                            df.srv[c][a:b].copy_(self.host_srv[c][a:b],
                                                 non_blocking=True)
                    _native.check(L.rlfc_copy2d(
                        rt.data_ptr() + lo * row_b, plane,
                        self.host_roots.data_ptr() + lo * row_b, plane,
                        (hi - lo) * row_b, nplanes, 0, s_in.cuda_stream),
                        "rlfc_copy2d")
                    ev = torch.cuda.Event()
                    ev.record(s_in)
                s_dec.wait_event(ev)
                y0 = lo * B - self.rows[0] * B
                y1 = min(hi * B, hdr.height) - self.rows[0] * B
                dst = self.out.data_ptr() + y0 * W * 3
                rc = _native.RLFC_ERR_ARGUMENT
                if ws is not None:
                    rc = L.rlfc_decode_field_staged(
                        df.ref, 0, None, lo, hi, dst, img, W * 3,
                        ws[0].data_ptr(), ws[1], ws[2], ws[3], None, 0,
                        self.status.data_ptr(), s_dec.cuda_stream)
                if rc == _native.RLFC_ERR_ARGUMENT:
                    rc = L.rlfc_decode_field(
                        df.ref, 0, None, lo, hi, dst, img, W * 3,
                        self.status.data_ptr(), s_dec.cuda_stream)
                _native.check(rc, "rlfc_decode_field")
                ev2 = torch.cuda.Event()
                ev2.record(s_dec)
                s_out.wait_event(ev2)
                if y1 > y0:
                    _native.check(L.rlfc_copy2d(
                        self.out_host.data_ptr() + y0 * W * 3, img,
                        self.out.data_ptr() + y0 * W * 3, img,
                        (y1 - y0) * W * 3, hdr.s_count * hdr.t_count, 1,
                        s_out.cuda_stream), "rlfc_copy2d")
        s_out.synchronize()
        s_dec.synchronize()
        _raise_word(self.status.cpu().item())
        return self.out_host
