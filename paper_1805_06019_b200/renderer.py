"""Novel-view synthesis on the B200: drop-in for the reference rlfc.renderer.

`render_view` keeps the reference signature (renderer.py:279-305).  A view is
rendered in two device steps: the fused decode kernel writes the pose's tap
cameras (<= 4 for a slab pose) as RGB8 into HBM, then one render kernel
evaluates every output pixel with the reference's float64 arithmetic in the
reference's operation order (bit-exact; rlfc_render.cu).  `render_views`
batches many poses: the union of their tap cameras is decoded once and every
view is rendered from it in one launch.

Per-frame constants that the reference computes with numpy (pinhole basis,
renderer.py:190-209) are computed here with the same numpy expressions, so
they are identical to the reference's bit for bit.
"""

import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _native, colorspace, decoder
from .lightfield import PlaneGeometry, default_geometry

SNAP_EPS = 1e-9


@dataclass(frozen=True)
class LfCoord:
    s: float
    t: float
    u: float
    v: float


@dataclass(frozen=True)
class SlabPose:
    """Eye on the camera plane at grid position (s, t); focal_z refocuses."""
    s: float
    t: float
    width: int
    height: int
    focal_z: float = None


@dataclass(frozen=True)
class CameraPose:
    """Free pinhole camera: eye point, look direction, vertical fov."""
    eye: tuple
    look: tuple
    fov_deg: float
    width: int
    height: int

    def __post_init__(self):
        if self.fov_deg <= 0 or self.fov_deg >= 180:
            raise ValueError("fov must be in (0, 180)")
        if all(abs(v) < 1e-12 for v in self.look):
            raise ValueError("look direction is zero")


@dataclass(frozen=True)
class GridInfo:
    xs: np.ndarray
    ys: np.ndarray
    width: int
    height: int


def grid_info_for(state) -> GridInfo:
    hdr = state.header
    return GridInfo(xs=np.arange(hdr.s_count, dtype=np.float64),
                    ys=np.arange(hdr.t_count, dtype=np.float64),
                    width=hdr.width, height=hdr.height)


def _snap(f):
    r = round(f)
    return float(r) if abs(f - r) < SNAP_EPS else float(f)


def _axis_taps(coord, count):
    """[(index, weight)] with zero weights dropped (renderer.py:119-131)."""
    c = min(max(coord, 0.0), float(count - 1))
    if count == 1:
        return [(0, 1.0)]
    i0 = min(int(math.floor(c)), count - 2)
    f = _snap(c - i0)
    taps = []
    if f < 1.0:
        taps.append((i0, 1.0 - f))
    if f > 0.0:
        taps.append((i0 + 1, f))
    return taps


def ray_to_lf_coords(ray, geometry: PlaneGeometry, grid):
    """Fractional (s, t, u, v) of one ray, or None outside the slab."""
    origin, direction = (np.asarray(v, dtype=np.float64) for v in ray)
    if abs(direction[2]) < 1e-15:
        raise ValueError("ray parallel to the light-slab planes")
    if not isinstance(grid, GridInfo):
        grid = GridInfo(xs=grid.camera_positions[:, 0, 0].astype(np.float64),
                        ys=grid.camera_positions[0, :, 1].astype(np.float64),
                        width=grid.width, height=grid.height)
    tc = (geometry.camera_plane_z - origin[2]) / direction[2]
    cx = origin[0] + tc * direction[0]
    cy = origin[1] + tc * direction[1]
    if not (grid.xs[0] <= cx <= grid.xs[-1] and
            grid.ys[0] <= cy <= grid.ys[-1]):
        return None
    s = float(np.interp(cx, grid.xs, np.arange(len(grid.xs))))
    t = float(np.interp(cy, grid.ys, np.arange(len(grid.ys))))
    ti = (geometry.image_plane_z - origin[2]) / direction[2]
    ix = origin[0] + ti * direction[0]
    iy = origin[1] + ti * direction[1]
    x0, y0, x1, y1 = geometry.image_plane_extent
    if not (x0 <= ix <= x1 and y0 <= iy <= y1):
        return None
    u = (ix - x0) / (x1 - x0) * grid.width - 0.5
    v = (iy - y0) / (y1 - y0) * grid.height - 0.5
    return LfCoord(_snap(s), _snap(t), _snap(u), _snap(v))


def _block_rgb(state, s, t, bx, by, stop_level, memo):
    key = (s, t, bx, by, stop_level)
    if memo is not None and key in memo:
        return memo[key]
    blocks, _ = decoder.decode_blocks(
        state, [(s, t, bx, by, c, stop_level) for c in range(3)])
    planes = blocks.cpu().numpy()
    rgb = np.stack(colorspace.ycocgr_to_rgb(*planes)).clip(0, 255) \
        .astype(np.float64)
    if memo is not None:
        memo[key] = rgb
    return rgb


def sample_quadrilinear(state, coord: LfCoord, stop_level=0, memo=None):
    """16-tap blend around coord (renderer.py:147-169); GPU block decodes."""
    hdr = state.header
    b = hdr.block_size
    acc = np.zeros(3)
    for s, ws in _axis_taps(coord.s, hdr.s_count):
        for t, wt in _axis_taps(coord.t, hdr.t_count):
            for u, wu in _axis_taps(coord.u, hdr.width):
                for v, wv in _axis_taps(coord.v, hdr.height):
                    rgb = _block_rgb(state, s, t, u // b, v // b, stop_level,
                                     memo)
                    acc += (ws * wt * wu * wv) * rgb[:, v % b, u % b]
    return np.floor(acc + 0.5).clip(0, 255).astype(np.uint8)


def _slab_rays(pose: SlabPose, geometry, grid: GridInfo):
    """Eye and per-pixel directions (renderer.py:172-187; host reference)."""
    focal = pose.focal_z if pose.focal_z is not None else \
        geometry.image_plane_z
    if focal == geometry.camera_plane_z:
        raise ValueError("focal plane coincides with the camera plane")
    ex = float(np.interp(pose.s, np.arange(len(grid.xs)), grid.xs))
    ey = float(np.interp(pose.t, np.arange(len(grid.ys)), grid.ys))
    eye = np.array([ex, ey, geometry.camera_plane_z])
    x0, y0, x1, y1 = geometry.image_plane_extent
    tx = x0 + (np.arange(pose.width) + 0.5) * (x1 - x0) / pose.width
    ty = y0 + (np.arange(pose.height) + 0.5) * (y1 - y0) / pose.height
    targets = np.zeros((pose.height, pose.width, 3))
    targets[:, :, 0] = tx[None, :]
    targets[:, :, 1] = ty[:, None]
    targets[:, :, 2] = focal
    return eye, targets - eye


def _pinhole_basis(pose: CameraPose, geometry):
    """Per-frame eye / look / right / down / tan(fov/2) / aspect, computed
    with the reference's numpy expressions (renderer.py:190-209)."""
    eye = np.asarray(pose.eye, dtype=np.float64)
    if abs(eye[2] - geometry.image_plane_z) < 1e-12:
        raise ValueError("eye lies on the image plane")
    look = np.asarray(pose.look, dtype=np.float64)
    look = look / np.linalg.norm(look)
    up = np.array([0.0, 1.0, 0.0])
    if abs(np.dot(up, look)) > 1.0 - 1e-9:
        up = np.array([1.0, 0.0, 0.0])
    right = np.cross(look, up)
    right /= np.linalg.norm(right)
    down = np.cross(look, right)
    half = math.tan(math.radians(pose.fov_deg) / 2.0)
    aspect = pose.width / pose.height
    return np.concatenate([eye, look, right, down, [half, aspect]])


def _snap_v(f):
    r = np.rint(f)
    return np.where(np.abs(f - r) < SNAP_EPS, r, f)


def _axis_taps_v(coord, count):
    """_axis_taps over an array: (i0, has_lo, has_hi) with the reference's
    clamping and snapping (renderer.py:119-131)."""
    c = np.minimum(np.maximum(coord, 0.0), float(count - 1))
    if count == 1:
        z = np.zeros(c.shape, dtype=np.int64)
        return z, np.ones(c.shape, bool), np.zeros(c.shape, bool)
    i0 = np.minimum(np.floor(c).astype(np.int64), count - 2)
    f = _snap_v(c - i0)
    return i0, f < 1.0, f > 0.0


def _pinhole_first_failure(state, pose, geometry, stop_level):
    """Raise what the reference's render_view raises for this pinhole pose on
    a stream with corrupt records (renderer.py:295-305): pixels in raster
    order, each pixel's taps in (s, t, u, v) order, blocks decoded once
    (memo) with channels 0, 1, 2; the first failing block raises
    FormatError, a ray parallel to the slab raises ValueError where the
    reference reaches it.  Error path only: ray coordinates are evaluated with
    the reference's numpy expressions over all pixels, the touched blocks
    decoded in one batch on the GPU."""
    hdr = state.header
    b = hdr.block_size
    S, T, W, H = hdr.s_count, hdr.t_count, hdr.width, hdr.height
    eye = np.asarray(pose.eye, dtype=np.float64)
    fr = _pinhole_basis(pose, geometry)
    look, right, down, half, aspect = fr[3:6], fr[6:9], fr[9:12], fr[12], fr[13]
    px = (np.arange(pose.width) + 0.5) / pose.width * 2.0 - 1.0
    py = (np.arange(pose.height) + 0.5) / pose.height * 2.0 - 1.0
    dirs = (look[None, None, :] + (px[None, :, None] * half * aspect) * right[None, None, :]
            + (py[:, None, None] * half) * down[None, None, :]).reshape(-1, 3)
    dz = dirs[:, 2]
    parallel = np.abs(dz) < 1e-15
    first_par = int(np.argmax(parallel)) if parallel.any() else None
    with np.errstate(divide="ignore", invalid="ignore"):
        tc = (geometry.camera_plane_z - eye[2]) / dz
        cx, cy = eye[0] + tc * dirs[:, 0], eye[1] + tc * dirs[:, 1]
        ti = (geometry.image_plane_z - eye[2]) / dz
        ix, iy = eye[0] + ti * dirs[:, 0], eye[1] + ti * dirs[:, 1]
    xs = np.arange(S, dtype=np.float64)
    ys = np.arange(T, dtype=np.float64)
    x0, y0, x1, y1 = geometry.image_plane_extent
    hit = ((xs[0] <= cx) & (cx <= xs[-1]) & (ys[0] <= cy) & (cy <= ys[-1]) &
           (x0 <= ix) & (ix <= x1) & (y0 <= iy) & (iy <= y1) & ~parallel)
    idx = np.flatnonzero(hit)
    sc = _snap_v(np.interp(cx[idx], xs, np.arange(S)))
    tcoord = _snap_v(np.interp(cy[idx], ys, np.arange(T)))
    u = _snap_v((ix[idx] - x0) / (x1 - x0) * W - 0.5)
    v = _snap_v((iy[idx] - y0) / (y1 - y0) * H - 0.5)
    taps = [_axis_taps_v(sc, S), _axis_taps_v(tcoord, T), _axis_taps_v(u, W), _axis_taps_v(v, H)]
    keys, order = [], []
    for a in range(2):
        for bb in range(2):
            for cc in range(2):
                for dd in range(2):
                    ok = np.ones(idx.shape, bool)
                    coord = []
                    for ax, sel in zip(taps, (a, bb, cc, dd)):
                        i0, lo, hi = ax
                        ok &= lo if sel == 0 else hi
                        coord.append(i0 + sel)
                    ss, tt, uu, vv = coord
                    key = ((ss * T + tt) * hdr.block_grid[1] + vv // b) * hdr.block_grid[0] + uu // b
                    keys.append(np.where(ok, key, -1))
                    order.append(idx * 16 + ((a * 2 + bb) * 2 + cc) * 2 + dd)
    keys = np.stack(keys, 1).ravel()
    order = np.stack(order, 1).ravel()
    valid = keys >= 0
    keys, order = keys[valid], order[valid]
    srt = np.argsort(order, kind="stable")
    keys, order = keys[srt], order[srt]
    uk, first = np.unique(keys, return_index=True)
    wb, hb = hdr.block_grid
    bx = uk % wb
    byy = (uk // wb) % hb
    cam = uk // (wb * hb)
    req = np.stack([np.repeat(cam // T, 3), np.repeat(cam % T, 3), np.repeat(bx, 3), np.repeat(byy, 3),
                    np.tile(np.arange(3), len(uk)), np.full(3 * len(uk), stop_level)], 1).astype(np.int32)
    fail_pix = None
    if len(req):
        _, st = decoder.decode_blocks(state, req, raise_errors=False)
        st = np.asarray(st.cpu().numpy() if hasattr(st, "cpu") else st).reshape(-1, 3)
        bad = np.flatnonzero((st != 0).any(1))
        if len(bad):
            j = bad[np.argmin(first[bad])]
            fail_pix = int(order[first[j]]) // 16
            code = int(st[j][np.flatnonzero(st[j])[0]])
    if first_par is not None and (fail_pix is None or first_par <= fail_pix):
        raise ValueError("ray parallel to the light-slab planes")
    if fail_pix is not None:
        decoder._raise_status(code)


def _geom_struct(geometry):
    x0, y0, x1, y1 = geometry.image_plane_extent
    return (geometry.camera_plane_z, geometry.image_plane_z, x0, y0, x1, y1)


def render_views(state, poses, stop_level=0, geometry=None,
                 background=(0, 0, 0), device=None, out=None, _host=None):
    """Render a batch of same-size poses; returns a CUDA uint8 tensor
    (n, height, width, 3).  geometry / background: one for all poses or one
    per pose."""
    import torch
    hdr = state.header
    decoder._check_level(state, stop_level)
    poses = list(poses)
    n = len(poses)
    if n == 0:
        raise ValueError("no poses")
    kinds = {type(p) for p in poses}
    for k in kinds:
        if k not in (SlabPose, CameraPose):
            raise TypeError(f"unknown pose type {k.__name__}")
    if len(kinds) != 1:
        raise TypeError("a batch must hold one pose type")
    ow, oh = poses[0].width, poses[0].height
    if any((p.width, p.height) != (ow, oh) for p in poses):
        raise ValueError("a batch must share one output size")
    S, T, W, H = hdr.s_count, hdr.t_count, hdr.width, hdr.height
    per_pose = isinstance(geometry, (list, tuple)) and geometry and \
        isinstance(geometry[0], (PlaneGeometry, type(None)))
    if per_pose:
        geos = [default_geometry(S, T) if g is None else g for g in geometry]
        gstruct = np.array([_geom_struct(g) for g in geos], dtype=np.float64)
    else:
        one = default_geometry(S, T) if geometry is None else geometry
        geos = None
        gstruct = np.empty((n, 6), dtype=np.float64)
        gstruct[:] = _geom_struct(one)
    bgs = np.asarray(background, dtype=np.uint8).reshape(-1, 3)
    if bgs.shape[0] == 1 and n > 1:
        bgs = np.repeat(bgs, n, axis=0)
    df = decoder._field_on(state, device)
    dev = df.device
    L = _native.lib()
    stream = torch._C._cuda_getCurrentRawStream(dev.index)
    if out is None:
        out = torch.empty((n, oh, ow, 3), dtype=torch.uint8, device=dev)
    if kinds == {SlabPose}:
        pose_arr = np.array([(p.s, p.t, float(p.focal_z is not None),
                              float(p.focal_z or 0.0)) for p in poses],
                            dtype=np.float64)
        # renderer.py:175-176: a focal plane on the camera plane is rejected
        if n <= 8:
            bad = any((p.focal_z if p.focal_z is not None else g[1]) == g[0]
                      for p, g in zip(poses, gstruct.tolist()))
        else:
            focal = np.where(pose_arr[:, 2] != 0.0, pose_arr[:, 3], gstruct[:, 1])
            bad = bool(np.any(focal == gstruct[:, 0]))
        if bad:
            raise ValueError("focal plane coincides with the camera plane")
        return _render_slab_batch(state, df, stop_level, pose_arr, gstruct,
                                  np.ascontiguousarray(bgs, dtype=np.uint8),
                                  ow, oh, out, stream, _host)
    d_geom = torch.from_numpy(gstruct).to(dev)
    d_bg = torch.from_numpy(bgs).to(dev)
    if geos is None:
        geos = [one] * n
    frames = np.stack([_pinhole_basis(p, g) for p, g in zip(poses, geos)])
    d_frames = torch.from_numpy(np.ascontiguousarray(frames)).to(dev)
    need = torch.zeros(S * T, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _native.check(L.rlfc_render_pinhole_needs(
            S, T, W, H, d_frames.data_ptr(), d_geom.data_ptr(), n, ow, oh,
            need.data_ptr(), stream), "rlfc_render_pinhole_needs")
    cams = np.flatnonzero(need.cpu().numpy())
    field, slots, dstatus = _decode_cameras(state, cams, stop_level, device)
    if dstatus is not None and dstatus.cpu().item() != 0:
        # a tap camera holds a corrupt record; the reference decodes only the
        # blocks its rays sample (memoised decode_block_progressive), so it
        # raises only when one of those fails -- decide exactly that
        for p, g in zip(poses, geos):
            _pinhole_first_failure(state, p, g, stop_level)
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _native.check(L.rlfc_render_pinhole(
            field.data_ptr(), slots.data_ptr(), S, T, W, H,
            d_frames.data_ptr(), d_geom.data_ptr(), d_bg.data_ptr(), n, ow,
            oh, out.data_ptr(), status.data_ptr(), stream),
            "rlfc_render_pinhole")
    if (status.cpu().numpy() == -2).any():
        raise ValueError("ray parallel to the light-slab planes")
    return out


class _Staging:
    """Per-thread, per-device staging buffers of rlfc_render_slab_batch: one
    pinned host buffer and one device buffer (grown on demand)."""

    def __init__(self, dev):
        self.dev = dev
        self.cap = 0

    def buffers(self, nbytes):
        import torch
        if nbytes > self.cap:
            cap = max(4096, 1 << (nbytes - 1).bit_length())
            self.host = torch.empty(cap, dtype=torch.uint8).pin_memory()
            self.devbuf = torch.empty(cap, dtype=torch.uint8, device=self.dev)
            self.status = np.zeros(1, dtype=np.uint64)
            self.cap = cap
        return self.host, self.devbuf


_tls = threading.local()


def _staging(dev):
    d = getattr(_tls, "staging", None)
    if d is None:
        d = _tls.staging = {}
    st = d.get(dev.index)
    if st is None:
        st = d[dev.index] = _Staging(dev)
    return st


# tap-camera fields up to this size stay allocated on their DeviceField
# between batch calls: the calls on one field run under its enqueue lock and
# return drained, so the next call may reuse the scratch
_FIELD_KEEP_BYTES = 64 << 20


def _camera_field(df, shape):
    """The decoded tap cameras' scratch (caller holds df.enqueue_lock)."""
    import torch
    f = getattr(df, "render_field", None)
    if f is not None and tuple(f.shape) == shape:
        return f
    f = torch.empty(shape, dtype=torch.uint8, device=df.device)
    if shape[0] * shape[1] * shape[2] * shape[3] <= _FIELD_KEEP_BYTES:
        df.render_field = f
    return f


def _render_slab_batch(state, df, stop_level, pose_arr, gstruct, bgs, ow, oh,
                       out, stream, out_host=None):
    """Every slab pose of the batch in one native call
    (rlfc_render_slab_batch): tap cameras decoded by the staged path in slot
    mode, then one k_render_slab launch."""
    import torch
    hdr = state.header
    n = pose_arr.shape[0]
    L = _native.lib()
    nbytes = int(L.rlfc_render_staging_bytes(df.ref, n))
    stg = _staging(df.device)
    host, dbuf = stg.buffers(nbytes)
    shape = (min(hdr.s_count * hdr.t_count, 4 * n), hdr.height, hdr.width, 3)
    switch = decoder._get_device() != df.device.index
    if switch:
        prev = torch.cuda.current_device()
        torch.cuda.set_device(df.device)
    try:
        ws = df.staged_workspace(stream)
        args = (None, 0, 0, 0) if ws is None else (ws[0].data_ptr(), ws[1], ws[2], ws[3])
        with df.enqueue_lock:
            field = _camera_field(df, shape)
            rc = L.rlfc_render_slab_batch(
                df.ref, stop_level, *args, pose_arr.ctypes.data, gstruct.ctypes.data, bgs.ctypes.data, n, ow,
                oh, field.data_ptr(), field.shape[0], out.data_ptr(), host.data_ptr(), dbuf.data_ptr(),
                stg.cap, None if out_host is None else out_host.data_ptr(), stg.status.ctypes.data, stream)
    finally:
        if switch:
            torch.cuda.set_device(prev)
    _native.check(rc, "rlfc_render_slab_batch")
    decoder._raise_word(int(stg.status[0]))
    return out


def _decode_cameras(state, cams, stop_level, device):
    """Decode the given cameras (serial indices s*T + t) into a compact
    field; returns (field, slots, status word tensor or None)."""
    import torch
    hdr = state.header
    S, T = hdr.s_count, hdr.t_count
    df = state.device_field(device)
    cams = np.asarray(cams, dtype=np.int64)
    slots = np.full(S * T, -1, dtype=np.int32)
    slots[cams] = np.arange(len(cams), dtype=np.int32)
    d_slots = torch.from_numpy(slots).to(df.device)
    if len(cams):
        field, status = decoder.decode_field_slots(state, stop_level, d_slots,
                                                   len(cams), device=device,
                                                   rows=cams % T)
        return field, d_slots, status
    field = torch.zeros((1, hdr.height, hdr.width, 3), dtype=torch.uint8,
                        device=df.device)
    return field, d_slots, None


def render_view(state, pose, stop_level=0, geometry: PlaneGeometry = None,
                background=(0, 0, 0)):
    """Render one view as uint8 RGB (reference renderer.py:279-305)."""
    if not isinstance(pose, (SlabPose, CameraPose)):
        raise TypeError(f"unknown pose type {type(pose).__name__}")
    if isinstance(pose, SlabPose):
        # the native batch call also brings the view back into a pinned
        # array the result owns (one stream drain per call)
        import torch
        host = torch.empty((1, pose.height, pose.width, 3), dtype=torch.uint8, pin_memory=True)
        render_views(state, [pose], stop_level, geometry, background, _host=host)
        return host.numpy()[0]
    return decoder._to_host(render_views(state, [pose], stop_level, geometry,
                                         background)[0])
