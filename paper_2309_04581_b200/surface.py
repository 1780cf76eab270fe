"""Meshes and BSDF records mirroring `hybridrt.surface`
(reference `pkg/src/hybridrt/surface.py:35-188`).

These are plain host-side records. Intersection and BSDF sampling run on
the GPU (`csrc/bvh.cuh`, `csrc/shade.cuh`); the BVH itself is built by the
native library at `hrt_create` time, so there is no Python BVH here.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field
from typing import Optional

import numpy as np

from .core import Transform, vec3

MAT_LAMBERTIAN = 0
MAT_MIRROR = 1
MAT_DIELECTRIC = 2


def _spectrum01(c, what):
    c = vec3(c)
    if (c < 0).any() or (c > 1).any():
        raise ValueError(f"{what} channels must lie in [0, 1], got {c}")
    return c


@dataclass
class Lambertian:
    albedo: np.ndarray

    def __post_init__(self):
        self.albedo = _spectrum01(self.albedo, "albedo")


@dataclass
class Mirror:
    reflectance: np.ndarray

    def __post_init__(self):
        self.reflectance = _spectrum01(self.reflectance, "reflectance")


@dataclass
class Dielectric:
    ior: float
    tint: np.ndarray = dc_field(default_factory=lambda: np.ones(3))

    def __post_init__(self):
        if not self.ior > 0:
            raise ValueError(f"ior must be > 0, got {self.ior}")
        self.tint = _spectrum01(self.tint, "tint")


def material_record(bsdf):
    """(kind, rgb, ior) for the GPU material table; duck-typed by class name
    so reference `hybridrt.surface` BSDF objects pack the same way."""
    kind = type(bsdf).__name__
    if kind == "Lambertian":
        return MAT_LAMBERTIAN, np.asarray(bsdf.albedo, np.float64), 1.0
    if kind == "Mirror":
        return MAT_MIRROR, np.asarray(bsdf.reflectance, np.float64), 1.0
    if kind == "Dielectric":
        return MAT_DIELECTRIC, np.asarray(bsdf.tint, np.float64), float(bsdf.ior)
    raise TypeError(f"unknown bsdf {type(bsdf)}")


def face_normals_of(vertices: np.ndarray, indices: np.ndarray, name="mesh") -> np.ndarray:
    """Unit geometric normals cross(v1-v0, v2-v0)/|.| in the reference's
    float64 operation order (surface.py:169-176)."""
    tri = vertices[indices]
    e1 = tri[:, 1] - tri[:, 0]
    e2 = tri[:, 2] - tri[:, 0]
    n = np.empty_like(e1)
    n[:, 0] = e1[:, 1] * e2[:, 2] - e1[:, 2] * e2[:, 1]
    n[:, 1] = e1[:, 2] * e2[:, 0] - e1[:, 0] * e2[:, 2]
    n[:, 2] = e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]
    length = np.sqrt((n[:, 0] * n[:, 0] + n[:, 1] * n[:, 1]) + n[:, 2] * n[:, 2])
    scale = max(float(np.abs(vertices).max()), 1.0) if len(vertices) else 1.0
    if (length < 1e-12 * scale * scale).any():
        raise ValueError(f"mesh '{name}': degenerate zero-area triangle")
    return n / length[:, None]


class TriangleMesh:
    """Indexed world-space triangles, one BSDF, optional per-face emission."""

    def __init__(self, vertices, indices, bsdf, emission=None,
                 world_from_object: Optional[Transform] = None, name: str = "mesh"):
        self.name = name
        verts = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        idx = np.asarray(indices, dtype=np.int64).reshape(-1, 3)
        if idx.size and (idx.min() < 0 or idx.max() >= len(verts)):
            raise ValueError(f"mesh '{name}': face index out of range")
        self.world_from_object = world_from_object or Transform.identity()
        self.vertices = self.world_from_object.point(verts) if world_from_object else verts
        self.indices = idx
        self.bsdf = bsdf
        self.face_normals = face_normals_of(self.vertices, self.indices, name)
        if emission is not None:
            emission = np.asarray(emission, dtype=np.float64)
            if emission.ndim == 1:
                emission = np.broadcast_to(emission, (len(idx), 3)).copy()
            if emission.shape != (len(idx), 3) or (emission < 0).any():
                raise ValueError(f"mesh '{name}': emission must be (faces, 3) and >= 0")
        self.emission = emission

    def recompute_normals(self):
        self.face_normals = face_normals_of(self.vertices, self.indices, self.name)

    def triangle_vertices(self) -> np.ndarray:
        return self.vertices[self.indices]

    @property
    def is_emissive(self) -> bool:
        return self.emission is not None and bool((self.emission > 0).any())
