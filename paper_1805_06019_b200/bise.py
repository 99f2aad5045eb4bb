"""Bounded-integer-sequence coding: the canonical range table and helpers.

The table is part of the stream format (reference bise.py:22-60): a block's
one-byte descriptor indexes it.  Entry d has cardinality N = 2^b (plain bit
fields), 3*2^b (base-3 pack of up to 5 high digits in 8 bits + low bits) or
5*2^b (base-5 pack of up to 3 digits in 7 bits + low bits).

Decoding of coded payloads runs on the GPU (librlfc_b200.so
`rlfc_bise_decode`, replacing kernels.bise_decode_core); encoding belongs to
the stream producer (paper_1805_06019_b200.producer).
"""

from dataclasses import dataclass

import numpy as np

from .errors import FormatError

MODE_BITS, MODE_TRIT, MODE_QUINT = 0, 1, 2

RANGE_CARDINALITIES = tuple(
    base << b for b in range(12) for base in (1, 3, 5)
    if 2 <= (base << b) <= 2048)
RANGE_CARDINALITIES = tuple(sorted(set(RANGE_CARDINALITIES)))
assert len(RANGE_CARDINALITIES) == 30
MAX_VALUE = RANGE_CARDINALITIES[-1] - 1


@dataclass(frozen=True)
class RangeDescriptor:
    """One row of the canonical range table."""
    table_index: int
    mode: int
    low_bits: int
    cardinality: int


def _split(n):
    b = (n & -n).bit_length() - 1
    return {1: MODE_BITS, 3: MODE_TRIT, 5: MODE_QUINT}[n >> b], b


RANGE_TABLE = tuple(RangeDescriptor(i, *_split(n), n)
                    for i, n in enumerate(RANGE_CARDINALITIES))
TABLE_MODE = np.array([r.mode for r in RANGE_TABLE], dtype=np.uint8)
TABLE_BITS = np.array([r.low_bits for r in RANGE_TABLE], dtype=np.uint8)


def payload_bits(mode, bits, count):
    """Exact unpadded bit length of `count` coded values (kernels.py:63-70)."""
    if mode == MODE_BITS:
        return count * bits
    if mode == MODE_TRIT:
        return 8 * -(-count // 5) + count * bits
    return 7 * -(-count // 3) + count * bits


def payload_size(rng: RangeDescriptor, count):
    if count < 0:
        raise ValueError("count must be non-negative")
    return payload_bits(rng.mode, rng.low_bits, count)


def payload_bytes_table(count):
    """Padded payload bytes per descriptor for `count` values."""
    return np.array([(payload_size(r, count) + 7) // 8 for r in RANGE_TABLE],
                    dtype=np.int64)


def zigzag(v):
    """0, -1, 1, -2, 2 -> 0, 1, 2, 3, 4 (arrays accepted)."""
    v = np.asarray(v, dtype=np.int64)
    return np.where(v < 0, -2 * v - 1, 2 * v).astype(np.uint32)


def unzigzag(z):
    """Inverse of zigzag (arrays accepted)."""
    z = np.asarray(z, dtype=np.int64)
    return np.where(z & 1, -((z + 1) >> 1), z >> 1).astype(np.int64)


def select_range(max_value):
    """Smallest table entry whose cardinality exceeds max_value."""
    if max_value < 0:
        raise ValueError("max_value must be unsigned")
    if max_value > MAX_VALUE:
        raise FormatError(
            f"value {max_value} exceeds the range table (max {MAX_VALUE})")
    idx = int(np.searchsorted(np.asarray(RANGE_CARDINALITIES), max_value,
                              side="right"))
    return RANGE_TABLE[idx]


def bise_encode(values, rng: RangeDescriptor) -> bytes:
    """Pack values (< rng.cardinality) into a byte-padded string (host)."""
    from . import producer
    return producer.bise_encode(values, rng)


def bise_decode(data, count, rng: RangeDescriptor) -> np.ndarray:
    """Decode `count` values of one payload on the GPU (bise.py:108-118)."""
    raw = bytes(data)
    need = (payload_size(rng, count) + 7) // 8
    if len(raw) < need:
        raise FormatError(f"payload truncated: {len(raw)} bytes, need {need}")
    from .decoder import bise_decode_batch
    vals, status = bise_decode_batch([raw], [rng.table_index], count)
    if int(status[0]) != 0:
        raise FormatError("corrupt pack byte in coded stream")
    return vals[0]
