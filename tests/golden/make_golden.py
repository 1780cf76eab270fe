"""Generate tests/golden/*.npz by running the REAL reference package
(`hybridrt`, imported from /root/reference/pkg/src) in the build container.

The fixtures travel to the GPU box (where /root/reference does not exist) and
pin both the CPU oracle (tests/test_golden.py, not gpu) and the CUDA path
(tests/test_gpu_golden.py) to the reference's own outputs:

  rng.npz     rng.uniform on 20,000 random key tuples           (rng.py:54-57)
  rays.npz    _sample_jitter + Camera.primary_rays, 3 cameras   (render.py:61-74, 320-330)
  bvh.npz     Bvh.intersect_batch / any_hit_batch, 2 meshes      (surface.py:377-478)
  field.npz   RadianceGrid.sample_batch incl. outside / borders  (field.py:143-161)
  images.npz  finalize -> encode_ppm / encode_pfm bytes of 3 HDR frames incl. the sRGB
              cut, the 1.0 rail, > 1, zeros and tiny values   (render.py:399-401, images.py:37-64)
  transport.npz  emitters.build_transport (per-face transport operator) of a Lambertian
              room with an emissive quad, 2 poses, 4 spp, max_depth 3  (emitters.py:73-166)
  render.npz  render / render_surface_only / render_volume_only on dense-grid scenes
              (mirror fog, glass fog, Lambertian room, shadowed slab), with every
              input array needed to rebuild the scenes without the reference.

Run: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
"""

import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hybridrt import assets, rng  # noqa: E402
from hybridrt.core import Transform  # noqa: E402
from hybridrt.field import RadianceGrid  # noqa: E402
from hybridrt.images import HdrImage  # noqa: E402
from hybridrt.render import finalize  # noqa: E402
from hybridrt.emitters import build_transport  # noqa: E402
from hybridrt.render import (Camera, EmitterSet, _sample_jitter, render,  # noqa: E402
                             render_surface_only, render_volume_only)
from hybridrt.scene import CameraConfig, RenderConfig, Scene, SceneConfig, scene_diagonal  # noqa: E402
from hybridrt.surface import Bvh, Dielectric, Lambertian, Mirror, TriangleMesh  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def make_scene(field=None, meshes=(), emitters=None, camera=None, **kw):
    meshes = list(meshes)
    camera = camera or Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(30), (8, 8))
    cfg = SceneConfig(camera=CameraConfig(position=[0, 0, 3], look_at=[0, 0, 0],
                                          resolution=list(camera.resolution)))
    return Scene(config=cfg, camera=camera, render=RenderConfig(**kw), field=field, meshes=meshes,
                 bvh=Bvh(meshes), blocker_bvh=Bvh([m for m in meshes if not m.is_emissive]),
                 emitters=emitters, collider_sdfs=[],
                 spawn_eps=1e-4 * scene_diagonal(field, meshes))


def gen_rng():
    g = np.random.default_rng(7)
    n = 20000
    keys = np.stack([g.integers(-2**40, 2**40, n), g.integers(0, 2**31, n), g.integers(0, 64, n),
                     g.integers(0, 9, n), g.integers(0, 9, n), g.integers(0, 1100, n)], 1)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), keys=keys, u=rng.uniform(*keys.T))


def gen_rays():
    cams = [(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(40), (64, 64), 1, 0),
            (Transform.look_at([2.5, 1.0, 3.0], [0, 0.2, 0]), math.radians(40), (80, 60), 16, 3),
            (Transform.look_at([0.3, -2, 1.5], [0, 0.2, -1]), math.radians(63), (37, 23), 8, 11)]
    out = {}
    for i, (pose, fov, res, spp, seed) in enumerate(cams):
        cam = Camera(pose, fov, res)
        w, h = res
        pix = np.repeat(np.arange(w * h), spp)
        smp = np.tile(np.arange(spp), w * h)
        jx, jy = _sample_jitter(seed, pix, smp, spp)
        o, d = cam.primary_rays(pix, jx, jy)
        out.update({f"c{i}_m": pose.m, f"c{i}_fov": fov, f"c{i}_res": np.array(res),
                    f"c{i}_spp": spp, f"c{i}_seed": seed, f"c{i}_o": o, f"c{i}_d": d})
    np.savez_compressed(os.path.join(OUT, "rays.npz"), **out)


def gen_bvh():
    g = np.random.default_rng(3)
    v1, f1 = assets.icosphere(0.5, 3)
    v2, f2 = assets.box((-1.2, -0.8, -0.5), (1.1, 0.9, 0.7))
    meshes = [TriangleMesh(v1, f1, Dielectric(1.5)), TriangleMesh(v2, f2, Lambertian(np.full(3, .5)))]
    bvh = Bvh(meshes)
    n = 20000
    o = g.normal(size=(n, 3))
    o = 3.0 * o / np.linalg.norm(o, axis=1, keepdims=True)
    o[: n // 4] = g.uniform(-0.4, 0.4, (n // 4, 3))
    d = g.uniform(-0.8, 0.8, (n, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, f = bvh.intersect_batch(o, d)
    tmin = g.uniform(0, 0.5, n)
    tmax = tmin + g.uniform(0, 3.0, n)
    anyh = bvh.any_hit_batch(o, d, tmin, tmax)
    np.savez_compressed(os.path.join(OUT, "bvh.npz"), v1=v1, f1=f1, v2=v2, f2=f2, o=o, d=d, t=t,
                        face=f, tmin=tmin, tmax=tmax, any_hit=anyh,
                        normals=bvh.face_normal, tri=bvh.tri)


def gen_field():
    g = np.random.default_rng(5)
    sig = g.uniform(0.0, 2.0, (7, 5, 6))
    rad = g.uniform(0.0, 1.0, (7, 5, 6, 3))
    grid = RadianceGrid((-1.0, -0.5, -1.5), (1.0, 1.5, 1.0), sig, rad)
    p = g.uniform(-1.6, 1.6, (5000, 3))
    p[:4] = [[-1.0, -0.5, -1.5], [1.0, 1.5, 1.0], [0.0, 1.5, -1.5], [1.0000001, 0, 0]]
    s, r = grid.sample_batch(p)
    np.savez_compressed(os.path.join(OUT, "field.npz"), lo=grid.bbox_lo, hi=grid.bbox_hi,
                        sigma=sig, radiance=rad, p=p, s=s, r=r)


def dense_field(seed):
    g = np.random.default_rng(seed)
    return g.uniform(0.5, 1.5, (8, 9, 10)), g.uniform(0, 1, (8, 9, 10, 3))



def gen_images():
    g = np.random.default_rng(5)
    frames = [g.uniform(0.0, 1.0, (9, 13, 3)),
              np.exp(g.normal(-2.0, 2.0, (16, 16, 3))),                  # HDR, spans 1e-4 .. 50
              np.zeros((4, 5, 3))]
    special = np.array([0.0, 0.0031308, np.nextafter(0.0031308, 1), 1.0, np.nextafter(1.0, 0),
                        1.5, 1e-300, 5e-324, 0.5, 0.21404114048223255, 1e6, 0.99999])
    frames[2].reshape(-1)[:len(special)] = special
    out = {}
    for i, f in enumerate(frames):
        img = HdrImage(f)
        out[f"px{i}"] = f
        out[f"ppm{i}"] = np.frombuffer(finalize(img, False), np.uint8)
        out[f"pfm{i}"] = np.frombuffer(finalize(img, True), np.uint8)
    np.savez_compressed(os.path.join(OUT, "images.npz"), **out)


def gen_transport():
    bv, bf = assets.box((-2, -2, -2), (2, 2, 2), inward=True)
    qv, qf = assets.quad((-1, -1, -1.9), (2, 0, 0), (0, 2, 0))
    cv, cf = assets.box((-0.5, -1.5, -1.0), (0.3, -0.4, 0.2))
    room = [TriangleMesh(bv, bf, Lambertian(np.full(3, 0.6))),
            TriangleMesh(qv, qf, Lambertian(np.array((0.2, 0.3, 0.4))), emission=np.array((3.0, 2.0, 1.0))),
            TriangleMesh(cv, cf, Lambertian(np.array((0.7, 0.5, 0.3))))]
    poses = [Camera(Transform.look_at([0, 0, 1.5], [0, 0, -1]), math.radians(60), (12, 10)),
             Camera(Transform.look_at([1.2, 0.8, 1.0], [0, -0.5, -1]), math.radians(50), (12, 10))]
    sc = make_scene(meshes=room, camera=poses[0], spp=4, seed=9, n_bounces=8)
    op = build_transport(sc, poses, max_depth=3)
    np.savez_compressed(os.path.join(OUT, "transport.npz"), a=op.a, bv=bv, bf=bf, qv=qv, qf=qf,
                        cv=cv, cf=cf)

def gen_render():
    out = {}
    v, f = assets.icosphere(0.4, 2)
    cam = Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(40), (32, 32))
    step = 3 * math.sqrt(3) / 256
    for name, seed, bsdf, nb in (("mirror", 0, Mirror(np.full(3, 0.9)), 2),
                                 ("glass", 1, Dielectric(1.5), 4)):
        sig, rad = dense_field(seed)
        sc = make_scene(field=RadianceGrid((-1.5,) * 3, (1.5,) * 3, sig, rad),
                        meshes=[TriangleMesh(v, f, bsdf)], camera=cam, spp=1, n_bounces=nb,
                        march_step=step)
        out[f"{name}_img"] = render(sc, spp=1, seed=0).pixels
        out[f"{name}_sigma"], out[f"{name}_rad"] = sig, rad
    out["ico_v"], out["ico_f"] = v, f
    # Lambertian room, constant fog, 4 spp stratified (render.py:325-329)
    bv, bf = assets.box((-2, -2, -2), (2, 2, 2), inward=True)
    qv, qf = assets.quad((-1, -1, -1.9), (2, 0, 0), (0, 2, 0))
    room = [TriangleMesh(bv, bf, Lambertian(np.full(3, 0.6))),
            TriangleMesh(qv, qf, Lambertian(np.zeros(3)), emission=np.array((3.0, 2.0, 1.0)))]
    cam2 = Camera(Transform.look_at([0, 0, 1.5], [0, 0, -1]), math.radians(60), (24, 24))
    sc = make_scene(field=RadianceGrid.constant((-2,) * 3, (2,) * 3, 0.3, (0.2, 0.1, 0.0)),
                    meshes=room, camera=cam2, spp=4, seed=5, n_bounces=6)
    out["room_img"] = render(sc).pixels
    out["room_surface_img"] = render_surface_only(sc).pixels
    out["room_bv"], out["room_bf"], out["room_qv"], out["room_qf"] = bv, bf, qv, qf
    # shadowed slab (reference tests/test_render.py:120-147 semantics)
    sv, sf = assets.quad((-4, -4, 3.0), (8, 0, 0), (0, 8, 0))
    cam3 = Camera(Transform.look_at([0, 0, -3], [0, 0, 0]), math.radians(25), (8, 8))
    for tag, r in (("07", 0.7), ("00", 0.0)):
        em = EmitterSet([[[-1, -1, 6], [1, -1, 6], [0, 1, 6]]], [r])
        sc = make_scene(field=RadianceGrid.constant((-1,) * 3, (1,) * 3, 1.0, (1, 1, 1)),
                        meshes=[TriangleMesh(sv, sf, Lambertian(np.full(3, 0.5)))], emitters=em,
                        camera=cam3, march_step=0.02, spp=4, seed=9)
        out[f"shadow{tag}_img"] = render(sc).pixels
    out["shadow_v"], out["shadow_f"] = sv, sf
    sig, rad = dense_field(2)
    sc = make_scene(field=RadianceGrid((-1.5,) * 3, (1.5,) * 3, sig, rad),
                    meshes=[TriangleMesh(v, f, Dielectric(1.5))], camera=cam, spp=2, n_bounces=4,
                    march_step=0.05)
    out["volume_img"] = render_volume_only(sc, spp=2, seed=3).pixels
    out["volume_sigma"], out["volume_rad"] = sig, rad
    np.savez_compressed(os.path.join(OUT, "render.npz"), **out)


if __name__ == "__main__":
    gen_rng()
    gen_rays()
    gen_bvh()
    gen_field()
    gen_images()
    gen_transport()
    gen_render()
    for fn in sorted(os.listdir(OUT)):
        if fn.endswith(".npz"):
            print(fn, os.path.getsize(os.path.join(OUT, fn)))
