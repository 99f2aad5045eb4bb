"""Compression front end: light field in, canonical .rlfc stream out.

Same parameters and report as the reference encoder (hierarchy.py:31-79,
encoder.py:13-57).  The work runs in the native producer (producer.py,
librlfc_producer.so), which reproduces the reference's RKV/SRV trees and
serialisation byte for byte and is parallel across cameras and blocks.
"""

import time
from dataclasses import dataclass, field

VALID_BLOCK_SIZES = (2, 4, 8, 16)
ROOT_CODECS = ("raw", "png", "jpeg2000")


@dataclass(frozen=True)
class FilterSpec:
    """Cluster filter: uniform, or Gaussian falloff (sigma in 1/256 steps)."""
    kind: str = "gaussian"
    sigma: float = 0.7

    def __post_init__(self):
        if self.kind not in ("uniform", "gaussian"):
            raise ValueError(f"unknown filter kind {self.kind!r}")
        if self.kind == "gaussian" and self.sigma <= 0:
            raise ValueError("sigma must be positive")

    @property
    def sigma_fp(self) -> int:
        return int(round(self.sigma * 256.0))

    def quantized_sigma(self) -> float:
        return self.sigma_fp / 256.0


@dataclass(frozen=True)
class EncodingParams:
    tree_height: int = 3
    cluster_factor: int = 2
    block_size: int = 4
    pixel_threshold: int = 4
    block_threshold: int = 80
    quant_shift: int = 2
    filter: FilterSpec = field(default_factory=FilterSpec)
    root_codec: str = "png"

    def __post_init__(self):
        if self.tree_height < 1:
            raise ValueError("tree_height must be >= 1")
        if self.cluster_factor != 2:
            raise ValueError("only 2x2 clustering is supported")
        if self.block_size not in VALID_BLOCK_SIZES:
            raise ValueError(f"block_size must be one of {VALID_BLOCK_SIZES}")
        if not 0 <= self.quant_shift <= 8:
            raise ValueError("quant_shift must be in [0, 8]")
        if self.pixel_threshold < 0 or self.block_threshold < 0:
            raise ValueError("thresholds must be >= 0")
        if self.root_codec not in ROOT_CODECS:
            raise ValueError(f"root_codec must be one of {ROOT_CODECS}")


@dataclass(frozen=True)
class EncodeReport:
    stream_bytes: int
    bpp_total: float
    bpp_channels: tuple
    root_bytes: tuple
    present_blocks: tuple        # per tree level 0..h-1, channels summed
    encode_seconds: float


def compress(lf, params: EncodingParams = None, threads=0, device=None):
    """Encode a LightFieldGrid; returns (stream bytes, EncodeReport).

    device=None runs the native C++ producer on `threads` host threads;
    a CUDA device ("cuda", "cuda:1") builds the RKV/SRV trees and the
    records there (producer.encode_gpu).  Both are byte-identical to the
    reference encoder (tests/test_producer.py, tests/test_gpu_encoder.py)."""
    from . import producer
    from .container import parse_header
    params = params or EncodingParams()
    t0 = time.perf_counter()
    if device is None:
        stream, present = producer.encode(lf, params, threads=threads)
    else:
        stream, present = producer.encode_gpu(lf, params, device=device)
    elapsed = time.perf_counter() - t0
    pixels = lf.s_count * lf.t_count * lf.width * lf.height
    hdr = parse_header(stream)
    return stream, EncodeReport(
        stream_bytes=len(stream), bpp_total=8.0 * len(stream) / pixels,
        bpp_channels=tuple(8.0 * sum(sec) / pixels
                           for sec in hdr.section_lengths),
        root_bytes=tuple(sec[0] for sec in hdr.section_lengths),
        present_blocks=tuple(int(v) for v in present),
        encode_seconds=elapsed)
