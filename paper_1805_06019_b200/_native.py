"""ctypes binding of librlfc_b200.so (the C ABI in include/rlfc_b200.h).

The product path has no CPU fallback: if the CUDA library is missing, fails
to load, or no CUDA device is visible, every decode / render call raises
NativeUnavailable.
"""

import ctypes
import os

from ._build import CUDA_LIB

RLFC_OK = 0
RLFC_ERR_CORRUPT_PACK = 1
RLFC_ERR_BAD_DESCRIPTOR = 2
RLFC_ERR_ARGUMENT = 3
RLFC_ERR_CUDA = 4
MAX_LEVELS = 32
KEY_MAX = 1 << 60


class NativeUnavailable(RuntimeError):
    """The sm_100a extension (librlfc_b200.so) or a CUDA device is missing."""


class RlfcField(ctypes.Structure):
    """Mirror of `rlfc_field` (include/rlfc_b200.h)."""
    _fields_ = [(n, ctypes.c_int32) for n in (
        "s_count", "t_count", "width", "height", "block", "tree_height",
        "quant_shift", "m_nodes", "wp", "hp", "wb", "hb", "rsx", "rsy",
        "roots_i16", "bitmap_bytes", "tile_bytes_max", "_reserved")] + [
        ("level_base", ctypes.c_int32 * MAX_LEVELS),
        ("level_sx", ctypes.c_int32 * MAX_LEVELS),
        ("level_sy", ctypes.c_int32 * MAX_LEVELS),
        ("srv", ctypes.c_void_p * 3),
        ("offsets", ctypes.c_void_p * 3),
        ("srv_len", ctypes.c_uint64 * 3),
        ("roots", ctypes.c_void_p)]


class RenderGeom(ctypes.Structure):
    """Mirror of `rlfc_render_geom`."""
    _fields_ = [(n, ctypes.c_double) for n in
                ("cam_z", "img_z", "x0", "y0", "x1", "y1")]


class RlfcDir(ctypes.Structure):
    """Mirror of `rlfc_dir` (the device record directory)."""
    _fields_ = [("tw", ctypes.c_int32), ("nb", ctypes.c_int32),
                ("nchunks", ctypes.c_int32), ("rows", ctypes.c_int32),
                ("n_blobs", ctypes.c_int64), ("nrec", ctypes.c_int64),
                ("scratch_bytes", ctypes.c_uint64),
                ("root_rgb_bytes", ctypes.c_uint64),
                ("rgb_stride", ctypes.c_int32), ("n_flagged", ctypes.c_int32),
                ("blob_bytes", ctypes.c_uint64),
                ("scratch", ctypes.c_void_p), ("blob_off", ctypes.c_void_p),
                ("flagged", ctypes.c_void_p), ("root_rgb", ctypes.c_void_p),
                ("blobs", ctypes.c_void_p), ("tables", ctypes.c_void_p)]


DIR_TABLE_BYTES = 16384


_lib = None
_SIGS = {
    "rlfc_dir_plan": ["p", "p"],
    "rlfc_dir_size": ["p", "p", "p"],
    "rlfc_dir_build": ["p", "p", "p"],
    "rlfc_decode_field_dir": ["p", "p", "i", "i", "i", "p", "q", "q", "p",
                              "p"],
    "rlfc_decode_blocks": ["p", "p", "i", "p", "p", "p"],
    "rlfc_decode_block_sync": ["p", "i", "i", "i", "i", "i", "i", "p", "p",
                               "p"],
    "rlfc_decode_planes": ["p", "i", "p", "i", "p", "p", "p"],
    "rlfc_decode_field": ["p", "i", "p", "i", "i", "p", "q", "q", "p", "p"],
    "rlfc_decode_field_simple": ["p", "i", "p", "i", "i", "p", "q", "q", "p",
                                 "p"],
    "rlfc_count_present": ["p", "p", "p"],
    "rlfc_staged_prepare": ["p", "p", "u", "u", "p", "p"],
    "rlfc_decode_blocks_indexed": ["p", "p", "u", "u", "p", "i", "p", "p", "p"],
    "rlfc_decode_workspace_bytes": ["p", "u", "p"],
    "rlfc_decode_field_staged": ["p", "i", "p", "i", "i", "p", "q", "q", "p",
                                 "u", "u", "i", "p", "i", "p", "p"],
    "rlfc_bise_decode": ["p", "p", "p", "i", "i", "p", "p", "p"],
    "rlfc_block_server_request": ["p", "p", "i", "i", "i", "i", "i", "i", "u", "p", "p", "p"],
    "rlfc_staged_index_view": ["p", "p", "u", "u", "p"],
    "rlfc_block_server_call": ["p"],
    "rlfc_block_server_stop": ["p", "p"],
    "rlfc_chain_core_sync": ["p", "u", "u", "i", "i", "p", "i", "i", "p", "p"],
    "rlfc_chain_core": ["p", "u", "p", "i", "i", "i", "p", "i", "i", "p", "p",
                        "p"],
    "rlfc_plane_core": ["p", "u", "p", "i", "i", "i", "i", "p", "i", "i", "p",
                        "p", "p", "p"],
    "rlfc_render_slab_batch": ["p", "i", "p", "u", "u", "i", "p", "p", "p", "i", "i", "i", "p", "i", "p",
                               "p", "p", "u", "p", "p", "p"],
    "rlfc_render_staging_bytes": ["p", "i"],
    "rlfc_decode_plane_host": ["p", "i", "i", "i", "i", "p", "p", "p", "p", "p", "p", "p"],
    "rlfc_decode_image_host": ["p", "i", "p", "u", "u", "i", "i", "i", "p", "p", "p", "p", "u", "p", "p"],
    "rlfc_render_slab": ["p", "p", "i", "i", "i", "i", "p", "p", "p", "i",
                         "i", "i", "p", "p"],
    "rlfc_render_pinhole": ["p", "p", "i", "i", "i", "i", "p", "p", "p", "i",
                            "i", "i", "p", "p", "p"],
    "rlfc_render_pinhole_needs": ["i", "i", "i", "i", "p", "p", "i", "i", "i",
                                  "p", "p"],
    "rlfc_copy2d": ["p", "q", "p", "q", "q", "q", "i", "p"],
    "rlfc_png_unfilter": ["p", "q", "i", "i", "i", "p", "q", "p", "p"],
    "rlfc_enc_planes": ["p", "q", "i", "i", "i", "i", "p", "p"],
    "rlfc_enc_pyramid": ["p", "i", "i", "p", "i", "i", "p", "i", "i", "p"],
    "rlfc_enc_srv_level": ["p", "p", "i", "i", "i", "i", "i", "i", "i", "q",
                           "i", "i", "i", "p", "p", "p", "p", "p"],
    "rlfc_enc_record_sizes": ["p", "q", "i", "i", "p", "p"],
    "rlfc_enc_records": ["p", "p", "q", "i", "i", "p", "p", "p"],
    "rlfc_root_planes": ["p", "i", "i", "i", "i", "i", "i", "p", "p", "p"],
    "rlfc_version": ["p", "i"],
}
class IndexView(ctypes.Structure):
    """rlfc_index_view (include/rlfc_b200.h)."""
    _fields_ = [("bm", ctypes.c_void_p), ("rk", ctypes.c_void_p),
                ("rec_flag", ctypes.c_void_p), ("entries", ctypes.c_void_p),
                ("nrec", ctypes.c_int64), ("nwp", ctypes.c_int32),
                ("_pad", ctypes.c_int32), ("cap", ctypes.c_uint64)]


class BlockCall(ctypes.Structure):
    """rlfc_block_call (include/rlfc_b200.h)."""
    _fields_ = [("f", ctypes.c_void_p), ("mb", ctypes.c_void_p), ("index", ctypes.c_void_p),
                ("stream", ctypes.c_void_p), ("idle_ns", ctypes.c_uint64), ("out", ctypes.c_void_p),
                ("req", ctypes.c_int32 * 6), ("_pad", ctypes.c_int32 * 2)]


_CT = {"p": ctypes.c_void_p, "i": ctypes.c_int32, "q": ctypes.c_int64,
       "u": ctypes.c_uint64}
EXPORTS = tuple(_SIGS)
_RESTYPE = {"rlfc_render_staging_bytes": ctypes.c_uint64}


def load_library(path=CUDA_LIB):
    """dlopen the library and declare every exported entry point."""
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} not built: run `python -m paper_1805_06019_b200._build` "
            "(nvcc, sm_100a)")
    try:
        L = ctypes.CDLL(path)
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
    for name, sig in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
        fn.argtypes = [_CT[c] for c in sig]
    return L


def lib():
    """The loaded library; requires a visible CUDA device."""
    global _lib
    if _lib is None:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable(
                "no CUDA device visible: the RLFC B200 path has no CPU "
                "fallback")
        _lib = load_library()
    return _lib


def check(rc, what):
    if rc != RLFC_OK:
        raise RuntimeError(f"{what} failed with status {rc}")


def decode_status_word(word):
    """(key, code) of a device status word, or None for success."""
    word = int(word)
    if word == 0:
        return None
    return KEY_MAX - (word >> 2), word & 3
