"""The five BASELINE.json configurations as synthetic scenes (SURVEY
Appendix B; builder-chosen details pinned here with their seeds, P8/P11).

    cfg0  64x64, 1 spp, 2 bounces, mirror icosphere s2 r0.4, hash L8 F2 T2^12 16->128, occ 32^3
    cfg1  800x800, 1 spp, 4 bounces, glass icosphere s5 r0.5 (IOR 1.5), L16 F2 T2^19 16->2048,
          occ 128^3, cap 1024 samples/path, early-out / threshold 1e-4, 100 cameras
    cfg2  512x512, 16 spp, 3 bounces, Lambertian plane (0.7) + 50k-triangle blob, cfg1 network
    cfg3  1920x1080, 8 spp, 4 bounces, 200 icospheres s4 (1,024,000 tris), mixed materials,
          30 frames of seeded rigid motion (BVH refit per frame), cfg1 network
    cfg4  3840x2160, 64 spp, 6 bounces, L16 F4 T2^21 16->4096 softplus HDR, emissive quad
          (radiance 10, r_src 1) + shadow rays occluded by a 300k-triangle torus

Every parameter comes from `np.random.default_rng(seed)`; nothing is read
from disk.
"""

from __future__ import annotations

import math

import numpy as np

from . import assets
from .core import Transform
from .field import NeuralField
from .scene import Camera, EmitterSet, RenderConfig, Scene
from .surface import Dielectric, Lambertian, Mirror, TriangleMesh

MARCH_STEP = 3.0 * math.sqrt(3.0) / 256.0
BBOX = ((-1.5, -1.5, -1.5), (1.5, 1.5, 1.5))


def network(cfg: int) -> NeuralField:
    if cfg == 0:
        return NeuralField.random(0, n_levels=8, n_features=2, log2_table=12, n_min=16, n_max=128,
                                  occupancy_res=32)
    if cfg in (1, 2, 3):
        return NeuralField.random(1, n_levels=16, n_features=2, log2_table=19, n_min=16,
                                  n_max=2048, occupancy_res=128)
    if cfg == 4:
        return NeuralField.random(4, n_levels=16, n_features=4, log2_table=21, n_min=16,
                                  n_max=4096, out_activation="softplus", occupancy_res=128)
    raise ValueError(f"unknown config {cfg}")


def look_at_safe(pos, target=(0.0, 0.0, 0.0)):
    """look_at with up (0,1,0), falling back to (0,0,1) near the poles (P8)."""
    fwd = np.asarray(target, np.float64) - np.asarray(pos, np.float64)
    fwd /= np.linalg.norm(fwd)
    up = (0.0, 1.0, 0.0) if abs(fwd[1]) <= 0.99 else (0.0, 0.0, 1.0)
    return Transform.look_at(pos, target, up)


def cfg1_cameras(n=100, radius=4.0, res=(800, 800), fov_deg=40.0):
    rng = np.random.default_rng(1)
    cams = []
    for _ in range(n):
        p = rng.normal(size=3)
        p = radius * p / np.linalg.norm(p)
        cams.append(Camera(look_at_safe(p), math.radians(fov_deg), res))
    return cams


def _march(**kw):
    base = dict(march_step=MARCH_STEP, seed=0)
    base.update(kw)
    return RenderConfig(**base)


def cfg0(field=None):
    v, f = assets.icosphere(0.4, 2)
    mesh = TriangleMesh(v, f, Mirror(np.ones(3)), name="mirror_ico")
    cam = Camera(Transform.look_at((0, 0, 3), (0, 0, 0)), math.radians(40.0), (64, 64))
    return Scene(camera=cam, render=_march(spp=1, n_bounces=2), field=field or network(0),
                 meshes=[mesh])


def cfg1(field=None, camera_index=0):
    v, f = assets.icosphere(0.5, 5)
    mesh = TriangleMesh(v, f, Dielectric(1.5), name="glass_ico")
    cam = cfg1_cameras()[camera_index]
    return Scene(camera=cam, render=_march(spp=1, n_bounces=4, threshold=1e-4, sample_cap=1024,
                                           early_t=1e-4),
                 field=field or network(1), meshes=[mesh])


def cfg2(field=None):
    pv, pf = assets.quad((-1.5, -0.62, 1.5), (3.0, 0.0, 0.0), (0.0, 0.0, -3.0))
    plane = TriangleMesh(pv, pf, Lambertian(np.full(3, 0.7)), name="plane")
    bv, bf = assets.blob(2, radius=0.5)
    body = TriangleMesh(bv, bf, Lambertian(np.full(3, 0.7)), name="blob")
    cam = Camera(look_at_safe((0.0, 1.2, 3.6)), math.radians(40.0), (512, 512))
    return Scene(camera=cam, render=_march(spp=16, n_bounces=3, threshold=1e-4, sample_cap=1024,
                                           early_t=1e-4),
                 field=field or network(2), meshes=[plane, body])


def cfg3_layout(seed=3, n=200):
    rng = np.random.default_rng(seed)
    radii = rng.uniform(0.05, 0.2, n)
    centres = rng.uniform(-1.5, 1.5, (n, 3))
    kinds = rng.integers(0, 3, n)               # 0 mirror, 1 glass, 2 diffuse
    velocity = rng.normal(0.0, 0.02, (n, 3))    # per-frame rigid translation
    return radii, centres, kinds, velocity


def apply_rigid(v, m):
    """World points of object points v (n, 3) under a 3x4 world_from_object m,
    row r as ((m0*x + m1*y) + m2*z) + m3 - the order hrt_refit_rigid uses."""
    v = np.asarray(v, np.float64)
    return np.stack([((m[r, 0] * v[:, 0] + m[r, 1] * v[:, 1]) + m[r, 2] * v[:, 2]) + m[r, 3]
                     for r in range(3)], axis=1)


def cfg3_transforms(frame, layout=None):
    """(200, 3, 4) world_from_object of every sphere at `frame` (P11: scale by
    the radius, translate to centre + frame * velocity)."""
    radii, centres, _, vel = layout or cfg3_layout()
    xf = np.zeros((len(radii), 3, 4))
    for a in range(3):
        xf[:, a, a] = radii
    xf[:, :, 3] = centres + frame * vel
    return xf


def cfg3(field=None, frame=0, res=(1920, 1080)):
    radii, centres, kinds, vel = cfg3_layout()
    base_v, base_f = assets.icosphere(1.0, 4)
    xf = cfg3_transforms(frame)
    meshes = []
    for i in range(len(radii)):
        bsdf = (Mirror(np.full(3, 0.9)), Dielectric(1.5), Lambertian(np.full(3, 0.7)))[kinds[i]]
        meshes.append(TriangleMesh(apply_rigid(base_v, xf[i]), base_f, bsdf, name=f"ico{i}"))
    cam = Camera(look_at_safe((0.0, 0.4, 4.5)), math.radians(40.0), res)
    return Scene(camera=cam, render=_march(spp=8, n_bounces=4, threshold=1e-4, sample_cap=1024,
                                           early_t=1e-4),
                 field=field or network(3), meshes=meshes)


def cfg3_move(scene, frame):
    """Rigid motion of frame `frame` applied in place on the host (the
    renderer then refits from the world faces; hrt_refit_rigid does the same
    from cfg3_transforms without touching the host meshes)."""
    base_v, _ = assets.icosphere(1.0, 4)
    xf = cfg3_transforms(frame)
    for i, m in enumerate(scene.meshes):
        m.vertices = apply_rigid(base_v, xf[i])
        m.recompute_normals()
    scene.touch()


def cfg4(field=None, res=(3840, 2160)):
    lv, lf = assets.quad((-0.5, 2.0, -0.5), (1.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    # front side (u x v = -y) faces down into the scene
    light = TriangleMesh(lv, lf, Lambertian(np.zeros(3)), emission=np.full(3, 10.0), name="light")
    tv, tf = assets.torus(major=0.55, minor=0.18, nu=500, nv=300, seed=4, amplitude=0.03)
    tv = tv[:, [0, 2, 1]] + np.array([0.0, 1.1, 0.0])   # axis along y, above the field centre
    torus = TriangleMesh(tv, tf[:, ::-1].copy(), Lambertian(np.full(3, 0.5)), name="torus")
    em = EmitterSet(lv[lf].reshape(-1, 3, 3), [1.0, 1.0])
    cam = Camera(look_at_safe((0.0, 0.3, 4.0)), math.radians(40.0), res)
    return Scene(camera=cam, render=_march(spp=64, n_bounces=6, threshold=1e-4, sample_cap=1024,
                                           early_t=1e-4),
                 field=field or network(4), meshes=[light, torus], emitters=em)


BUILDERS = {0: cfg0, 1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4}
