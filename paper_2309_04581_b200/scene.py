"""Scene container, camera, emitters and render settings mirroring the
reference (`render.py:44-107` for `Camera`/`EmitterSet`, `scene.py:138-144`
for `RenderConfig`, `scene.py:459-499` for `Scene`/`scene_diagonal`).

`Scene` is duck-type compatible with `hybridrt.scene.Scene`: the renderer
reads only `camera`, `render`, `field`, `meshes`, `emitters` and
`spawn_eps`, so a reference scene object can be passed straight to
`paper_2309_04581_b200.render`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field
from typing import Optional

import numpy as np

from .core import Transform


@dataclass
class Camera:
    """Pinhole camera; `fov` is the vertical field of view in radians."""

    pose: Transform
    fov: float
    resolution: tuple

    def __post_init__(self):
        w, h = self.resolution
        if w < 1 or h < 1:
            raise ValueError(f"resolution must be positive, got {self.resolution}")
        if not 0 < self.fov < math.pi:
            raise ValueError(f"vertical fov must be in (0, pi), got {self.fov}")
        self.resolution = (int(w), int(h))


class EmitterSet:
    """Area-light triangles with r_src clipped to [0, 1] (render.py:77-107)."""

    def __init__(self, triangles, r_src):
        self.triangles = np.asarray(triangles, dtype=np.float64).reshape(-1, 3, 3)
        self.r_src = np.clip(np.asarray(r_src, dtype=np.float64).reshape(-1), 0.0, 1.0)
        if len(self.triangles) != len(self.r_src):
            raise ValueError("emitter triangle/intensity count mismatch")
        e1 = self.triangles[:, 1] - self.triangles[:, 0]
        e2 = self.triangles[:, 2] - self.triangles[:, 0]
        self.areas = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
        total = self.areas.sum()
        if len(self.areas) and total <= 0:
            raise ValueError("emitter set has zero total area")
        self.cdf = np.cumsum(self.areas) / total if len(self.areas) else np.zeros(0)

    def __len__(self):
        return len(self.triangles)


@dataclass
class RenderConfig:
    """Reference defaults (scene.py:138-144) plus the two march limits the
    NeRF configs add: `sample_cap` NeRF samples per path
    (0 = unlimited) and an in-march early-out when max(T_spec) < `early_t`
    (0 = off)."""

    spp: int = 16
    n_bounces: int = 8
    threshold: float = 1e-3
    march_step: float = 0.05
    seed: int = 0
    sample_cap: int = 0
    early_t: float = 0.0


def scene_diagonal(field, meshes) -> float:
    """Diagonal of field box corners (world) plus mesh vertices (scene.py:482-499)."""
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    if field is not None:
        lo_f, hi_f = field.bbox_lo, field.bbox_hi
        corners = np.array([[x, y, z] for x in (lo_f[0], hi_f[0])
                            for y in (lo_f[1], hi_f[1]) for z in (lo_f[2], hi_f[2])])
        wc = field.world_from_field.point(corners)
        lo, hi = np.minimum(lo, wc.min(0)), np.maximum(hi, wc.max(0))
    for m in meshes:
        if len(m.vertices):
            lo, hi = np.minimum(lo, m.vertices.min(0)), np.maximum(hi, m.vertices.max(0))
    if (hi < lo).any():
        return 1.0
    return max(float(np.linalg.norm(hi - lo)), 1e-6)


@dataclass
class Scene:
    """Render-ready scene; read-only during a render pass."""

    camera: Camera
    render: RenderConfig
    field: object = None
    meshes: list = dc_field(default_factory=list)
    emitters: Optional[EmitterSet] = None
    spawn_eps: float = None
    version: int = 0

    def __post_init__(self):
        if self.spawn_eps is None:
            self.spawn_eps = 1e-4 * scene_diagonal(self.field, self.meshes)

    def touch(self):
        """Mark geometry as changed (vertices moved): next render refits."""
        self.version += 1


def make_scene(field=None, meshes=(), emitters=None, camera=None, **render_kw) -> Scene:
    """Test/bench helper with the reference tests' defaults
    (reference tests/test_render.py:25-36)."""
    camera = camera or Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(30), (8, 8))
    return Scene(camera=camera, render=RenderConfig(**render_kw), field=field,
                 meshes=list(meshes), emitters=emitters)
