"""Rebuild the scenes of tests/golden/render.npz with this package's own
types (no reference import), so the GPU box can compare against the
reference's recorded outputs."""

import math
import os

import numpy as np

from paper_2309_04581_b200.core import Transform
from paper_2309_04581_b200.field import RadianceGrid
from paper_2309_04581_b200.scene import Camera, EmitterSet, make_scene
from paper_2309_04581_b200.surface import Dielectric, Lambertian, Mirror, TriangleMesh

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def render_scenes():
    """name -> (scene, spp, seed, mode, expected image)."""
    g = load("render.npz")
    v, f = g["ico_v"], g["ico_f"]
    cam = Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(40), (32, 32))
    step = 3 * math.sqrt(3) / 256
    out = {}
    for name, bsdf, nb in (("mirror", Mirror(np.full(3, 0.9)), 2), ("glass", Dielectric(1.5), 4)):
        field = RadianceGrid((-1.5,) * 3, (1.5,) * 3, g[f"{name}_sigma"], g[f"{name}_rad"])
        sc = make_scene(field=field, meshes=[TriangleMesh(v, f, bsdf)], camera=cam, spp=1,
                        n_bounces=nb, march_step=step)
        out[name] = (sc, 1, 0, "hybrid", g[f"{name}_img"])
    room = [TriangleMesh(g["room_bv"], g["room_bf"], Lambertian(np.full(3, 0.6))),
            TriangleMesh(g["room_qv"], g["room_qf"], Lambertian(np.zeros(3)),
                         emission=np.array((3.0, 2.0, 1.0)))]
    cam2 = Camera(Transform.look_at([0, 0, 1.5], [0, 0, -1]), math.radians(60), (24, 24))
    sc = make_scene(field=RadianceGrid.constant((-2,) * 3, (2,) * 3, 0.3, (0.2, 0.1, 0.0)),
                    meshes=room, camera=cam2, spp=4, seed=5, n_bounces=6)
    out["room"] = (sc, 4, 5, "hybrid", g["room_img"])
    out["room_surface"] = (sc, 4, 5, "surface", g["room_surface_img"])
    cam3 = Camera(Transform.look_at([0, 0, -3], [0, 0, 0]), math.radians(25), (8, 8))
    for tag, r in (("07", 0.7), ("00", 0.0)):
        em = EmitterSet([[[-1, -1, 6], [1, -1, 6], [0, 1, 6]]], [r])
        sc = make_scene(field=RadianceGrid.constant((-1,) * 3, (1,) * 3, 1.0, (1, 1, 1)),
                        meshes=[TriangleMesh(g["shadow_v"], g["shadow_f"], Lambertian(np.full(3, 0.5)))],
                        emitters=em, camera=cam3, march_step=0.02, spp=4, seed=9)
        out[f"shadow{tag}"] = (sc, 4, 9, "hybrid", g[f"shadow{tag}_img"])
    field = RadianceGrid((-1.5,) * 3, (1.5,) * 3, g["volume_sigma"], g["volume_rad"])
    sc = make_scene(field=field, meshes=[TriangleMesh(v, f, Dielectric(1.5))], camera=cam, spp=2,
                    n_bounces=4, march_step=0.05)
    out["volume"] = (sc, 2, 3, "volume", g["volume_img"])
    return out


def ray_cameras():
    g = load("rays.npz")
    cams = []
    for i in range(3):
        res = tuple(int(x) for x in g[f"c{i}_res"])
        cam = Camera(Transform(g[f"c{i}_m"]), float(g[f"c{i}_fov"]), res)
        cams.append((cam, int(g[f"c{i}_spp"]), int(g[f"c{i}_seed"]), g[f"c{i}_o"], g[f"c{i}_d"]))
    return cams


def bvh_meshes():
    g = load("bvh.npz")
    return [TriangleMesh(g["v1"], g["f1"], Dielectric(1.5)),
            TriangleMesh(g["v2"], g["f2"], Lambertian(np.full(3, 0.5)))], g
