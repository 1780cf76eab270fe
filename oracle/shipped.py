"""The reference renderer AS SHIPPED, timed on a cfg3-shaped crop (context
for bench.py's cpu_baseline; SURVEY §8d / BASELINE.md §3 "also report the
reference as shipped, with a dense-grid stand-in").

MEASUREMENT INFRASTRUCTURE ONLY (like the rest of oracle/): bench.py's CPU
legs are the only caller; the product never imports it.

The reference `hybridrt` (pure Python/NumPy, installed unmodified into
baseline/_ref with `pip install --no-index --no-deps --target baseline/_ref`,
or taken from /root/reference/pkg/src in the build container) has no neural
field, so the NeRF is replaced by the reference's own dense
`RadianceGrid` (`field.py:104-161`) filled with the same near-homogeneous fog
the random-init NeRF produces (sigma = exp(N(0, 0.05^2)), radiance ~ 0.5,
SURVEY F5). Geometry, materials, camera, spp and bounces are cfg3's
(`paper_2309_04581_b200.configs.cfg3`, frame 0), built with the reference's
`TriangleMesh` / `Bvh` / `Camera` / `RenderConfig`. Every tile runs the
reference's `_render_tile` body for a 16x16 pixel block: `_sample_jitter`
(`render.py:320-330`) -> `Camera.primary_rays` (`render.py:61-74`) ->
`_trace_batch_hybrid` (`render.py:204-246`), the same tracer `render()` uses.
Field evaluations are counted at the field seam (`sample_batch`, points
inside the box).
"""

from __future__ import annotations

import importlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TILE = 16


def import_reference():
    """The `hybridrt` package: baseline/_ref (travels to the GPU box), else
    the read-only source tree of the build container. None if neither."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "hybridrt")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import hybridrt  # noqa: F401
            return p
    return None


_SCENE = None


def build_scene(frame=0):
    """Reference Scene of cfg3's frame `frame` with a dense fog stand-in."""
    from hybridrt import field as rf
    rr = importlib.import_module("hybridrt.render")     # (the package re-exports render())
    rs = importlib.import_module("hybridrt.scene")
    from hybridrt import surface as sf
    from hybridrt.core import Transform

    from paper_2309_04581_b200 import assets, configs
    radii, centres, kinds, _ = configs.cfg3_layout()
    base_v, base_f = assets.icosphere(1.0, 4)
    xf = configs.cfg3_transforms(frame)
    meshes = []
    for i in range(len(radii)):
        bsdf = (sf.Mirror((0.9, 0.9, 0.9)), sf.Dielectric(1.5), sf.Lambertian((0.7, 0.7, 0.7)))[kinds[i]]
        meshes.append(sf.TriangleMesh(configs.apply_rigid(base_v, xf[i]), base_f, bsdf, name=f"ico{i}"))
    g = np.random.default_rng(3)
    res = (64, 64, 64)
    sigma = np.exp(g.normal(0.0, 0.05, res))
    rad = 1.0 / (1.0 + np.exp(-g.normal(0.0, 0.3, res + (3,))))
    grid = rf.RadianceGrid(configs.BBOX[0], configs.BBOX[1], sigma, rad)
    # cfg3's camera (configs.cfg3: look_at_safe((0, 0.4, 4.5)) -> up (0, 1, 0), 40 deg)
    camera = rr.Camera(Transform.look_at((0.0, 0.4, 4.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0)),
                       np.radians(40.0), (1920, 1080))
    render_cfg = rs.RenderConfig(spp=8, n_bounces=4, threshold=1e-4, march_step=configs.MARCH_STEP,
                                 seed=0)
    bvh = sf.Bvh(meshes)
    diag = rs.scene_diagonal(grid, meshes)
    # no emitters -> the blocker tree is never traversed (render.py:157): share the closest-hit tree
    return rs.Scene(config=None, camera=camera, render=render_cfg, field=grid, meshes=meshes,
                    bvh=bvh, blocker_bvh=bvh, emitters=None, collider_sdfs=[],
                    spawn_eps=1e-4 * diag)


def scene():
    global _SCENE
    if _SCENE is None:
        _SCENE = build_scene()
    return _SCENE


def tile_job(tile_index):
    """(field evaluations, paths) of one 16x16 x 8 spp tile through the
    reference tracer (runs in a forked worker that inherited `scene()`)."""
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    rr = importlib.import_module("hybridrt.render")
    sc = scene()
    w, h = sc.camera.resolution
    tx = w // TILE
    x0, y0 = (tile_index % tx) * TILE, (tile_index // tx) * TILE
    ys, xs = np.meshgrid(np.arange(y0, y0 + TILE), np.arange(x0, x0 + TILE), indexing="ij")
    pix = (ys * w + xs).reshape(-1)
    spp = sc.render.spp
    count = [0]
    orig = sc.field.sample_batch

    def counted(p):
        s, r = orig(p)
        count[0] += int(np.count_nonzero(s > 0.0))
        return s, r

    sc.field.sample_batch = counted
    try:
        pix_rep = np.repeat(pix, spp)
        smp_rep = np.tile(np.arange(spp), len(pix))
        jx, jy = rr._sample_jitter(sc.render.seed, pix_rep, smp_rep, spp)
        o, d = sc.camera.primary_rays(pix_rep, jx, jy)
        L = rr._trace_batch_hybrid(sc, o, d, pix_rep, smp_rep, sc.render.seed)
        assert np.all(np.isfinite(L))
    finally:
        sc.field.sample_batch = orig
    return count[0], len(pix_rep)
