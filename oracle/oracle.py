"""CPU oracle for the RLFC decode / render hot path -- TEST INFRASTRUCTURE ONLY.

Restates the reference stream parsing (pkg/src/rlfc/container.py) in numpy
and drives the plain-C restatement of the hot loops (oracle/rlfc_oracle.c,
kernels.py / decoder.py / renderer.py) through ctypes.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this
module; the product package never does.

Parity of the oracle itself is pinned by tests/test_oracle_golden.py against
fixtures generated from the live reference (tools/make_goldens.py).
"""

import ctypes
import io
import math
import os
import struct
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librlfc_oracle.so")

# container.py:46 header layout
_HEADER_FMT = "<4sBBBBHHHHBBHHI2x9I"
HEADER_SIZE = 64
CHANNEL_BIAS = (0, 256, 256)          # container.py:56
# bise.py:22-25
RANGE_CARDINALITIES = (2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64,
                       80, 96, 128, 160, 192, 256, 320, 384, 512, 640, 768,
                       1024, 1280, 1536, 2048)


class OracleFormatError(Exception):
    pass


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        i32 = ctypes.c_int
        f64 = ctypes.c_double
        L.orc_payload_bits.restype = ctypes.c_int64
        L.orc_payload_bits.argtypes = [i32, i32, ctypes.c_int64]
        L.orc_bise_decode.argtypes = [vp, i32, i32, i32, vp]
        L.orc_field_decode_all.argtypes = [vp, i32, vp, i32, vp]
        L.orc_field_plane.argtypes = [vp, i32, i32, i32, i32, vp]
        L.orc_field_block.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp]
        L.orc_render_slab.argtypes = [vp, i32, i32, i32, i32, vp, f64, f64,
                                      i32, i32, i32, f64, vp, vp]
        L.orc_render_pinhole.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp,
                                         vp, vp, vp, f64, f64, i32, i32, vp,
                                         vp]
        L.orc_render_slab_decoding.argtypes = [vp, vp, f64, f64, i32, i32, i32,
                                               f64, i32, vp, vp, vp]
        L.orc_nproc.restype = i32
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class _Field(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "s_count", "t_count", "width", "height", "block", "tree_height",
        "quant_shift", "m_nodes", "wp", "hp", "wb", "hb", "rsx", "rsy")] + [
        ("srv", ctypes.c_void_p * 3), ("offsets", ctypes.c_void_p * 3),
        ("roots", ctypes.c_void_p), ("chains", ctypes.c_void_p)]


class _Geom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("cam_z", "img_z", "x0", "y0", "x1", "y1")]


def level_dims(S, T, l):                       # container.py:102-104
    return -(-S // (1 << l)), -(-T // (1 << l))


def chains_for(S, T, h):                       # container.py:107-145
    counts = [level_dims(S, T, l)[0] * level_dims(S, T, l)[1]
              for l in range(h)]
    out = np.zeros((S, T, h), dtype=np.int64)
    for s in range(S):
        for t in range(T):
            idx = []
            for l in range(h - 1, -1, -1):
                sx, _ = level_dims(S, T, l)
                idx.append(sum(counts[l + 1:]) + (t >> l) * sx + (s >> l))
            out[s, t] = idx
    return out


def _decode_root(blob, codec, wp, hp):         # container.py:175-195
    if codec == 0:
        if len(blob) != wp * hp * 2:
            raise OracleFormatError("raw root length")
        return np.frombuffer(blob, dtype="<u2").reshape(hp, wp).astype(np.int64)
    from PIL import Image
    with Image.open(io.BytesIO(blob)) as im:
        arr = np.asarray(im)
    if arr.shape != (hp, wp):
        raise OracleFormatError("root dims")
    return arr.astype(np.int64)


class OracleState:
    """Parsed stream (decoder.py:31-48 init, restated)."""

    def __init__(self, data):
        data = bytes(data)
        if len(data) < HEADER_SIZE:
            raise OracleFormatError("short")
        f = struct.unpack(_HEADER_FMT, data[:HEADER_SIZE])
        (magic, version, codec, B, h, S, T, W, H, shift, _filt, _sig, _tp,
         _tb, *flat) = f
        if magic != b"RLFC" or version != 1:
            raise OracleFormatError("magic/version")
        self.data = data
        self.S, self.T, self.W, self.H = S, T, W, H
        self.B, self.h, self.shift, self.codec = B, h, shift, codec
        self.wp, self.hp = -(-W // B) * B, -(-H // B) * B
        self.wb, self.hb = self.wp // B, self.hp // B
        self.rsx, self.rsy = level_dims(S, T, h)
        self.m_nodes = sum(level_dims(S, T, l)[0] * level_dims(S, T, l)[1]
                           for l in range(h))
        secs = [(flat[3 * c], flat[3 * c + 1], flat[3 * c + 2])
                for c in range(3)]
        self.sections = secs
        pos = HEADER_SIZE
        roots = np.zeros((self.rsx, self.rsy, 3, self.hp, self.wp), np.int32)
        self.srv, self.offsets = [], []
        for c in range(3):
            rl, ol, sl = secs[c]
            p = pos
            for y in range(self.rsy):
                for x in range(self.rsx):
                    (n,) = struct.unpack("<I", data[p:p + 4])
                    p += 4
                    roots[x, y, c] = _decode_root(
                        data[p:p + n], codec, self.wp, self.hp) - CHANNEL_BIAS[c]
                    p += n
            self.offsets.append(np.frombuffer(
                data, dtype="<u8", count=self.wb * self.hb,
                offset=pos + rl).copy())
            self.srv.append(np.frombuffer(data, dtype=np.uint8, count=sl,
                                          offset=pos + rl + ol).copy())
            pos += rl + ol + sl
        if pos != len(data):
            raise OracleFormatError("length")
        self.roots = np.ascontiguousarray(roots)
        self.chains = chains_for(S, T, h)
        fs = _Field()
        for name in ("wp", "hp", "wb", "hb", "rsx", "rsy", "m_nodes"):
            setattr(fs, name, getattr(self, name))
        fs.s_count, fs.t_count, fs.width, fs.height = S, T, W, H
        fs.block, fs.tree_height, fs.quant_shift = B, h, shift
        for c in range(3):
            fs.srv[c] = self.srv[c].ctypes.data
            fs.offsets[c] = self.offsets[c].ctypes.data
        fs.roots = self.roots.ctypes.data
        fs.chains = self.chains.ctypes.data
        self._fs = fs

    # decoder.py:197-210
    def decode_all(self, stop_level=0, nthreads=0):
        out = np.zeros((self.S, self.T, self.H, self.W, 3), np.uint8)
        bad = np.zeros(1, np.int64)
        st = lib().orc_field_decode_all(ctypes.byref(self._fs), stop_level,
                                        _p(out), nthreads, _p(bad))
        return out, int(st)

    # decoder.py:165-184
    def decode_plane(self, s, t, c, stop_level=0):
        out = np.zeros((self.hp, self.wp), np.int32)
        st = lib().orc_field_plane(ctypes.byref(self._fs), s, t, c,
                                   stop_level, _p(out))
        return out, int(st)

    def decode_planes(self, stop_level=0):
        out = np.zeros((self.S, self.T, 3, self.hp, self.wp), np.int32)
        st = 0
        for s in range(self.S):
            for t in range(self.T):
                for c in range(3):
                    o, e = self.decode_plane(s, t, c, stop_level)
                    out[s, t, c] = o
                    st = st or e
        return out, st

    # decoder.py:81-106
    def decode_block(self, s, t, bx, by, c, stop_level=0):
        out = np.zeros((self.B, self.B), np.int32)
        st = lib().orc_field_block(ctypes.byref(self._fs), s, t, bx, by, c,
                                   stop_level, _p(out))
        return out, int(st)

    def _geom(self, geometry):
        if geometry is None:                    # lightfield.py:37-43
            geometry = (0.0, 1.0, (-1.5, -1.5, self.S - 1 + 1.5,
                                   self.T - 1 + 1.5))
        cz, iz, (x0, y0, x1, y1) = geometry
        return _Geom(cz, iz, x0, y0, x1, y1)

    # renderer.py:233-276
    def render_slab(self, s, t, width, height, focal_z=None, stop_level=0,
                    geometry=None, background=(0, 0, 0), field=None):
        if field is None:
            field, st = self.decode_all(stop_level)
            assert st == 0
        g = self._geom(geometry)
        out = np.zeros((height, width, 3), np.uint8)
        bg = np.asarray(background, np.uint8)
        rc = lib().orc_render_slab(
            _p(field), self.S, self.T, self.W, self.H, ctypes.byref(g),
            float(s), float(t), width, height, int(focal_z is not None),
            float(focal_z or 0.0), _p(bg), _p(out))
        if rc == -1:
            raise ValueError("focal plane coincides with the camera plane")
        return out

    # renderer.py:190-209 per-frame basis (numpy, as the reference)
    @staticmethod
    def pinhole_basis(eye, look, fov_deg, width, height):
        eye = np.asarray(eye, dtype=np.float64)
        look = np.asarray(look, dtype=np.float64)
        look = look / np.linalg.norm(look)
        up = np.array([0.0, 1.0, 0.0])
        if abs(np.dot(up, look)) > 1.0 - 1e-9:
            up = np.array([1.0, 0.0, 0.0])
        right = np.cross(look, up)
        right /= np.linalg.norm(right)
        down = np.cross(look, right)
        half = math.tan(math.radians(fov_deg) / 2.0)
        aspect = width / height
        return eye, look, right, down, half, aspect

    # renderer.py:295-305
    def render_pinhole(self, eye, look, fov_deg, width, height, stop_level=0,
                       geometry=None, background=(0, 0, 0), field=None):
        if field is None:
            field, st = self.decode_all(stop_level)
            assert st == 0
        g = self._geom(geometry)
        e, lk, rt, dn, half, aspect = self.pinhole_basis(eye, look, fov_deg,
                                                         width, height)
        if abs(e[2] - g.img_z) < 1e-12:
            raise ValueError("eye lies on the image plane")
        out = np.zeros((height, width, 3), np.uint8)
        bg = np.asarray(background, np.uint8)
        arrs = [np.ascontiguousarray(a, np.float64) for a in (e, lk, rt, dn)]
        rc = lib().orc_render_pinhole(
            _p(field), self.S, self.T, self.W, self.H, self.B,
            ctypes.byref(g), *[_p(a) for a in arrs], half, aspect, width,
            height, _p(bg), _p(out))
        if rc == -2:
            raise ValueError("ray parallel to the light-slab planes")
        return out

    # reference-faithful per-view render cost (decode taps, then blend)
    def render_slab_decoding(self, s, t, width, height, focal_z=None,
                             stop_level=0, scratch=None):
        if scratch is None:
            scratch = np.zeros((self.S, self.T, self.H, self.W, 3), np.uint8)
        g = self._geom(None)
        out = np.zeros((height, width, 3), np.uint8)
        bg = np.zeros(3, np.uint8)
        rc = lib().orc_render_slab_decoding(
            ctypes.byref(self._fs), ctypes.byref(g), float(s), float(t),
            width, height, int(focal_z is not None), float(focal_z or 0.0),
            stop_level, _p(bg), _p(out), _p(scratch))
        assert rc == 0
        return out


def bise_decode(data, count, desc):
    """kernels.py:128-159 via bise.py:108-118 (status, values)."""
    n = RANGE_CARDINALITIES[desc]
    bits = (n & -n).bit_length() - 1
    odd = n >> bits
    mode = {1: 0, 3: 1, 5: 2}[odd]
    buf = np.frombuffer(bytes(data), dtype=np.uint8).copy()
    out = np.zeros(count, np.uint32)
    st = lib().orc_bise_decode(_p(buf), count, mode, bits, _p(out))
    return int(st), out


def payload_bits(desc, count):
    n = RANGE_CARDINALITIES[desc]
    bits = (n & -n).bit_length() - 1
    mode = {1: 0, 3: 1, 5: 2}[n >> bits]
    return int(lib().orc_payload_bits(mode, bits, count))
