"""Two-plane light-field containers, slab geometry and synthetic scenes.

Same public types as the reference lightfield.py:24-83 / 197-203.
synthesize_lightfield runs in the native producer (producer.py), which
reproduces the reference's integer-hash value-noise scene bit-exactly
(lightfield.py:207-302) and is parallel over cameras.
"""

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class PlaneGeometry:
    """Parallel camera and image planes plus the image-plane window."""
    camera_plane_z: float
    image_plane_z: float
    image_plane_extent: tuple          # world (x0, y0, x1, y1)

    def __post_init__(self):
        if self.camera_plane_z == self.image_plane_z:
            raise ValueError("camera plane and image plane must be distinct")


def default_geometry(s_count, t_count):
    """Geometry used when a stream carries none (lightfield.py:37-43)."""
    return PlaneGeometry(0.0, 1.0, (-1.5, -1.5, s_count - 1 + 1.5,
                                    t_count - 1 + 1.5))


@dataclass
class LightFieldGrid:
    """rgb[s, t, y, x, channel] 8-bit samples plus camera positions."""
    s_count: int
    t_count: int
    width: int
    height: int
    rgb: np.ndarray
    camera_positions: np.ndarray
    geometry: PlaneGeometry

    def __post_init__(self):
        want = (self.s_count, self.t_count, self.height, self.width, 3)
        if self.rgb.shape != want:
            raise ValueError(f"plane array shape {self.rgb.shape} != {want}")
        if self.camera_positions.shape != (self.s_count, self.t_count, 2):
            raise ValueError("camera_positions must be one 2D point per cell")
        xs = self.camera_positions[:, :, 0]
        ys = self.camera_positions[:, :, 1]
        if self.s_count > 1 and not (np.diff(xs, axis=0) > 0).all():
            raise ValueError("camera x positions must increase along the s axis")
        if self.t_count > 1 and not (np.diff(ys, axis=1) > 0).all():
            raise ValueError("camera y positions must increase along the t axis")

    def _check_index(self, s, t):
        if not (0 <= s < self.s_count and 0 <= t < self.t_count):
            raise IndexError(f"camera index ({s}, {t}) outside "
                             f"{self.s_count}x{self.t_count} grid")

    def image(self, s, t):
        self._check_index(s, t)
        return self.rgb[s, t]

    def camera_position(self, s, t):
        self._check_index(s, t)
        return (float(self.camera_positions[s, t, 0]),
                float(self.camera_positions[s, t, 1]))


def grid_positions(s_count, t_count):
    pos = np.zeros((s_count, t_count, 2))
    pos[:, :, 0] = np.arange(s_count)[:, None]
    pos[:, :, 1] = np.arange(t_count)[None, :]
    return pos


@dataclass(frozen=True)
class SyntheticSpec:
    s_count: int = 8
    t_count: int = 8
    width: int = 64
    height: int = 64
    seed: int = 7


def synthesize_lightfield(spec: SyntheticSpec, threads=0) -> LightFieldGrid:
    """The reference's deterministic procedural scene (lightfield.py:245-302)."""
    from . import producer
    if spec.s_count < 1 or spec.t_count < 1:
        raise ValueError("grid dimensions must be at least 1x1")
    if spec.width < 2 or spec.height < 2:
        raise ValueError("image resolution too small")
    rgb = producer.synthesize(spec, threads=threads)
    return LightFieldGrid(spec.s_count, spec.t_count, spec.width, spec.height,
                          rgb, grid_positions(spec.s_count, spec.t_count),
                          default_geometry(spec.s_count, spec.t_count))
