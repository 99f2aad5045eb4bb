"""GPU drop-in for the reference's kernel module (INTEGRATION.md Route 2).

The reference selects its kernel backend at import (kernels.py:22-44) and
its decoder calls three entry points with host numpy buffers
(decoder.py:101-104, 179-182):

    decode_chain_core(srv, rec_off, m_nodes, bsq, targets, shift,
                      table_mode, table_bits, out, tmp) -> int
    decode_plane_core(srv, offsets, blocks_x, blocks_y, m_nodes, block,
                      targets, shift, table_mode, table_bits,
                      root_plane, out_plane) -> int
    bise_decode_core(data, count, mode, bits, out) -> int

This module keeps those signatures, argument meanings, return codes
(0 ok / 1 corrupt pack / 2 bad descriptor, kernels.py:165-171) and in/out
buffers, and runs them on the B200 through the C ABI (rlfc_chain_core,
rlfc_plane_core, rlfc_bise_decode in include/rlfc_b200.h).  The SRV section
a caller passes is a zero-copy view of its immutable stream bytes
(container.py:391-399), so its device copy is cached by buffer address.
`tmp` is the reference's scratch buffer; it is not written.

There is no CPU fallback: without the extension or a CUDA device every call
raises _native.NativeUnavailable.
"""

import threading
from collections import OrderedDict

import numpy as np

from . import _native
from .bise import RANGE_TABLE

MODE_BITS, MODE_TRIT, MODE_QUINT = 0, 1, 2     # kernels.py:17-19
_SRV_PAD = 32
_cache = OrderedDict()
_cache_lock = threading.Lock()
_CACHE_MAX = 8


def _torch():
    import torch
    return torch


def _device_bytes(buf):
    """Device copy (+ zero tail) of a host buffer, cached by address.  The
    cache entry holds the host array too, so its memory cannot be freed and
    reused by another buffer while the entry lives."""
    torch = _torch()
    a = np.asarray(buf)
    key = (a.__array_interface__["data"][0], a.nbytes, torch.cuda.current_device())
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            _cache.move_to_end(key)
            return hit[1]
    host = torch.zeros(a.nbytes + _SRV_PAD, dtype=torch.uint8)
    host[:a.nbytes] = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy())
    d = host.cuda()
    with _cache_lock:
        _cache[key] = (a, d)
        while len(_cache) > _CACHE_MAX:
            _cache.popitem(last=False)
    return d


def _check_tables(table_mode, table_bits):
    # the reference passes its own range table (bise.py:59-60); the device
    # kernels carry the same table, so a caller's must match it
    if len(table_mode) != len(RANGE_TABLE) or len(table_bits) != len(RANGE_TABLE):
        raise ValueError("range table differs from the format's")


_tls = threading.local()


def _pinned_io(n):
    """Per-thread pinned host buffer (int32[n]) the latency kernel reads and
    writes over unified addressing."""
    torch = _torch()
    buf = getattr(_tls, "io", None)
    if buf is None or buf.numel() < n:
        buf = torch.empty(max(n, 257), dtype=torch.int32).pin_memory()
        _tls.io = buf
    return buf


def decode_chain_core(srv, rec_off, m_nodes, bsq, targets, shift,
                      table_mode, table_bits, out, tmp):
    """kernels.py:162-216 on the GPU; out (int32[bsq], pre-filled with the
    root block) receives the dequantised target residuals.  One call is one
    request (decoder.py:101-104), so it takes the latency path: targets in
    the kernel parameters, the block in pinned host memory, the status word
    polled (rlfc_chain_core_sync)."""
    torch = _torch()
    L = _native.lib()
    _check_tables(table_mode, table_bits)
    dsrv = _device_bytes(srv)
    tg = np.ascontiguousarray(targets, dtype=np.int64)
    bsq = int(bsq)
    if tg.size <= 16:
        io = _pinned_io(bsq + 1)
        host = io.numpy()
        host[:bsq] = np.reshape(out, -1)
        _native.check(L.rlfc_chain_core_sync(dsrv.data_ptr(), np.asarray(srv).nbytes, int(rec_off),
                                             int(m_nodes), bsq, tg.ctypes.data, int(tg.size), int(shift),
                                             io.data_ptr(), torch.cuda.current_stream().cuda_stream),
                      "rlfc_chain_core_sync")
        out[...] = host[:bsq].reshape(np.shape(out))
        return int(host[bsq])
    dtg = torch.as_tensor(tg).cuda()
    offs = torch.tensor([int(rec_off)], dtype=torch.int64).cuda()
    acc = torch.as_tensor(np.ascontiguousarray(out, dtype=np.int32).reshape(-1)).cuda()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(L.rlfc_chain_core(dsrv.data_ptr(), np.asarray(srv).nbytes, offs.data_ptr(), 1, int(m_nodes),
                                    bsq, dtg.data_ptr(), int(dtg.numel()), int(shift), acc.data_ptr(),
                                    status.data_ptr(), torch.cuda.current_stream().cuda_stream),
                  "rlfc_chain_core")
    out[...] = acc.cpu().numpy().reshape(np.shape(out))
    return int(status.item())


def decode_plane_core(srv, offsets, blocks_x, blocks_y, m_nodes, block,
                      targets, shift, table_mode, table_bits,
                      root_plane, out_plane):
    """kernels.py:219-242 on the GPU: every block of one plane."""
    torch = _torch()
    L = _native.lib()
    _check_tables(table_mode, table_bits)
    dsrv = _device_bytes(srv)
    doffs = _device_bytes(np.asarray(offsets).view(np.uint8))
    tg = torch.as_tensor(np.ascontiguousarray(targets, dtype=np.int64)).cuda()
    root = torch.as_tensor(np.ascontiguousarray(root_plane, dtype=np.int32)).cuda()
    dout = torch.as_tensor(np.ascontiguousarray(out_plane, dtype=np.int32)).cuda()
    status = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    _native.check(L.rlfc_plane_core(dsrv.data_ptr(), np.asarray(srv).nbytes, doffs.data_ptr(), int(blocks_x),
                                    int(blocks_y), int(m_nodes), int(block), tg.data_ptr(), int(tg.numel()),
                                    int(shift), root.data_ptr(), dout.data_ptr(), status.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream), "rlfc_plane_core")
    out_plane[...] = dout.cpu().numpy()
    word = int(status.item()) & 0xFFFFFFFFFFFFFFFF
    return 0 if word == 0xFFFFFFFFFFFFFFFF else word & 3


def bise_decode_core(data, count, mode, bits, out):
    """kernels.py:128-159 on the GPU: count values into out (uint32)."""
    torch = _torch()
    L = _native.lib()
    desc = next((d for d, r in enumerate(RANGE_TABLE) if r.mode == mode and r.low_bits == bits), None)
    if desc is None:
        raise ValueError(f"no range with mode {mode} and {bits} low bits")
    raw = np.zeros(len(data) + _SRV_PAD, dtype=np.uint8)
    raw[:len(data)] = np.frombuffer(bytes(np.asarray(data, dtype=np.uint8)), dtype=np.uint8)
    d = torch.from_numpy(raw).cuda()
    offs = torch.zeros(1, dtype=torch.int64, device="cuda")
    descs = torch.tensor([desc], dtype=torch.uint8, device="cuda")
    vals = torch.zeros((1, int(count)), dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(L.rlfc_bise_decode(d.data_ptr(), offs.data_ptr(), descs.data_ptr(), 1, int(count),
                                     vals.data_ptr(), status.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream), "rlfc_bise_decode")
    out[:count] = vals.cpu().numpy().view(np.uint32)[0]
    return int(status.item())
