"""Live pinning of the CPU oracle against the real reference package
(imported from /root/reference in the build container; skipped elsewhere,
where tests/test_golden.py carries the recorded outputs instead)."""

import math

import numpy as np
import pytest

from oracle import rng as orng
from oracle import tracer
from oracle.field import dense_sample
from oracle.geometry import TriangleSet, moller_trumbore, ray_slab
from paper_2309_04581_b200.pack import pack_camera, pack_field, pack_scene

pytestmark = pytest.mark.reference


def _ref_scene(h, field=None, meshes=(), emitters=None, camera=None, **kw):
    from hybridrt.scene import CameraConfig, RenderConfig, Scene, SceneConfig, scene_diagonal
    from hybridrt.surface import Bvh
    meshes = list(meshes)
    cfg = SceneConfig(camera=CameraConfig(position=[0, 0, 3], look_at=[0, 0, 0],
                                          resolution=list(camera.resolution)))
    return Scene(config=cfg, camera=camera, render=RenderConfig(**kw), field=field, meshes=meshes,
                 bvh=Bvh(meshes), blocker_bvh=Bvh([m for m in meshes if not m.is_emissive]),
                 emitters=emitters, collider_sdfs=[],
                 spawn_eps=1e-4 * scene_diagonal(field, meshes))


def test_rng_broadcast_and_scalars(hybridrt, rng):
    from hybridrt import rng as href
    pix = rng.integers(0, 10**9, 5000)
    assert np.array_equal(orng.uniform(3, pix, 2, 1, orng.LIGHT_U, 5),
                          href.uniform(3, pix, 2, 1, href.LIGHT_U, 5))
    for keys in [(0, 0, 0, 0, 0, 0), (-5, 7, 1, 2, 3, 4), (2**62, 1, 1, 1, 8, 1023)]:
        assert orng.uniform(*keys) == href.uniform(*keys)


def test_primary_rays_random_cameras(hybridrt, rng):
    from hybridrt.core import Transform
    from hybridrt.render import Camera, _sample_jitter
    for _ in range(8):
        pos = rng.normal(size=3) * 3
        cam = Camera(Transform.look_at(pos, rng.normal(size=3) * 0.3),
                     rng.uniform(0.2, 2.5), (int(rng.integers(1, 40)), int(rng.integers(1, 40))))
        w, h = cam.resolution
        spp = int(rng.choice([1, 3, 4, 9]))
        pix = np.repeat(np.arange(w * h), spp)
        smp = np.tile(np.arange(spp), w * h)
        jx, jy = _sample_jitter(5, pix, smp, spp)
        ox, dx = cam.primary_rays(pix, jx, jy)
        ojx, ojy = tracer.sample_jitter(5, pix, smp, spp)
        assert np.array_equal(ojx, jx) and np.array_equal(ojy, jy)
        oo, od = tracer.primary_rays(pack_camera(cam), pix, jx, jy)
        assert np.array_equal(oo, ox)
        assert np.array_equal(od, dx)


def test_slab_and_moller_trumbore(hybridrt, rng):
    from hybridrt.field import _ray_slab
    from hybridrt.surface import _moller_trumbore
    o = rng.normal(size=(4000, 3)) * 2
    d = rng.normal(size=(4000, 3))
    d[:300, 0] = 0.0
    d[300:400, 1] = 0.0
    lo, hi = np.array([-1.0, -0.5, -2.0]), np.array([1.0, 1.5, 0.5])
    for a, b in zip(ray_slab(lo, hi, o, d), _ray_slab(lo, hi, o, d)):
        assert np.array_equal(a, b)
    tri = rng.normal(size=(50, 3, 3))
    e1, e2 = tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]
    args = (o[:, None], d[:, None], tri[None, :, 0], e1[None], e2[None], 0.0, np.inf)
    assert np.array_equal(moller_trumbore(*args), _moller_trumbore(*args))


def test_nearest_hit_equals_reference_bvh_on_soup(hybridrt, rng):
    from hybridrt.surface import Bvh, Lambertian, TriangleMesh
    tri = rng.uniform(-1, 1, (600, 1, 3)) + rng.normal(0, 0.2, (600, 3, 3))
    mesh = TriangleMesh(tri.reshape(-1, 3), np.arange(1800).reshape(-1, 3),
                        Lambertian(np.full(3, 0.5)))
    bvh = Bvh([mesh])
    o = rng.uniform(-2, 2, (5000, 3))
    d = rng.normal(size=(5000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t_ref, f_ref = bvh.intersect_batch(o, d)
    ts = TriangleSet(bvh.tri[:, 0], bvh.edge1, bvh.edge2)
    t, f = ts.nearest(o, d)
    assert np.array_equal(f, f_ref) and np.array_equal(t, t_ref)
    tb, fb = ts.brute_nearest(o, d)
    assert np.array_equal(fb, f_ref) and np.array_equal(tb, t_ref)
    tmin = rng.uniform(0, 1, 5000)
    tmax = tmin + rng.uniform(0, 2, 5000)
    assert np.array_equal(ts.any_hit(o, d, tmin, tmax), bvh.any_hit_batch(o, d, tmin, tmax))


def test_dense_field_plugin(hybridrt, rng):
    from hybridrt.core import Transform
    from hybridrt.field import RadianceGrid
    grid = RadianceGrid((-1, -1, -1), (1, 2, 1), rng.uniform(0, 3, (4, 6, 5)),
                        rng.uniform(0, 1, (4, 6, 5, 3)),
                        world_from_field=Transform.translate((0.2, -0.1, 0.3)))
    p = rng.uniform(-1.5, 2.5, (6000, 3))
    s_ref, r_ref = grid.sample_batch(p)
    s, r = dense_sample(pack_field(grid), p)
    assert np.array_equal(s, s_ref) and np.array_equal(r, r_ref)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_hybrid_scenes_bit_equal(hybridrt, seed):
    """Random dense fog + random mirror/glass/diffuse meshes + optional
    emitters: the oracle tracer equals hybridrt.render.render bit for bit."""
    from hybridrt import assets
    from hybridrt.core import Transform
    from hybridrt.field import RadianceGrid
    from hybridrt.render import Camera, EmitterSet, render
    from hybridrt.surface import Dielectric, Lambertian, Mirror, TriangleMesh
    g = np.random.default_rng(100 + seed)
    field = RadianceGrid((-1.2,) * 3, (1.2,) * 3, g.uniform(0, 2, (5, 6, 7)),
                         g.uniform(0, 1, (5, 6, 7, 3)))
    meshes = []
    for k in range(3):
        v, f = assets.icosphere(g.uniform(0.15, 0.4), 1, center=g.uniform(-0.6, 0.6, 3))
        bsdf = [Mirror(g.uniform(0.5, 1, 3)), Dielectric(g.uniform(1.2, 1.8)),
                Lambertian(g.uniform(0.2, 0.9, 3))][k]
        meshes.append(TriangleMesh(v, f, bsdf))
    qv, qf = assets.quad((-1, 1.1, -1), (2, 0, 0), (0, 0, 2))
    meshes.append(TriangleMesh(qv, qf[:, ::-1], Lambertian(np.zeros(3)), emission=np.full(3, 4.0)))
    em = EmitterSet(qv[qf].reshape(-1, 3, 3), [0.6, 0.6]) if seed != 1 else None
    cam = Camera(Transform.look_at(g.normal(size=3) * 0.5 + [0, 0, 3], [0, 0, 0]),
                 math.radians(45), (12, 10))
    scene = _ref_scene(hybridrt, field=field, meshes=meshes, emitters=em, camera=cam, spp=4,
                       seed=seed, n_bounces=5, march_step=0.08)
    want = render(scene).pixels
    got = tracer.render(pack_scene(scene), pack_camera(cam), 4, seed)
    assert np.array_equal(got, want)


def wide_frame_scene(h):
    """A frame wide enough that the reference traces a 16-row band in several
    batches of samples per pixel (render.py:339-349: 65536 // (16 * 512) = 8
    samples per batch at w = 512; the last band of 4 rows takes 32): a
    random dense grid in front of a tilted mirror quad."""
    from hybridrt.assets import quad
    from hybridrt.core import Transform
    from hybridrt.field import RadianceGrid
    from hybridrt.render import Camera
    from hybridrt.surface import Mirror, TriangleMesh
    g = np.random.default_rng(11)
    field = RadianceGrid((-1, -1, -1), (1, 1, 1), g.uniform(0, 1.5, (6, 6, 6)), g.uniform(0, 1, (6, 6, 6, 3)))
    v, f = quad((-3, -3, -1.5), (6, 0, 0.5), (0, 6, 0))
    cam = Camera(Transform.look_at((0, 0, 3), (0, 0, 0)), math.radians(30), (512, 20))
    return _ref_scene(h, field=field, meshes=[TriangleMesh(v, f, Mirror(np.full(3, 0.8)))], camera=cam,
                      spp=12, n_bounces=2, march_step=0.08, seed=4)


def test_render_batches_like_the_reference_on_wide_frames(hybridrt):
    """Per-pixel sums grouped as the reference's sample batches: bit-equal
    on a 512-wide frame at 12 spp (batches of 8 + 4 in full bands, 12 in
    the 4-row last band), where a plain sample-order sum differs in the
    last bits."""
    from hybridrt.render import render
    scene = wide_frame_scene(hybridrt)
    want = render(scene).pixels
    got = tracer.render(pack_scene(scene), pack_camera(scene.camera), 12, 4)
    assert np.array_equal(got, want)
