"""GPU parity: the sm_100a kernels (through the C ABI, libhrt.so) against the
CPU oracle on identical seeded inputs.

Bar (BASELINE north star): RNG draws, camera rays, BVH face ids, hash
indices/features, occupancy bits and evaluated-sample sets bit-exact;
deterministic images within 1e-3 max abs per channel (here far tighter for
dense-grid scenes, which are float64 end to end).
"""

import math

import numpy as np
import pytest
import torch

from oracle import rng as orng
from oracle import tracer
from oracle.field import build_occupancy, neural_encode, neural_mlp, occupancy_bits
from oracle.geometry import TriangleSet
from paper_2309_04581_b200 import assets, configs
from paper_2309_04581_b200.core import Transform
from paper_2309_04581_b200.field import NeuralField, RadianceGrid
from paper_2309_04581_b200.pack import pack_camera, pack_scene
from paper_2309_04581_b200.renderer import Renderer, primary_rays, uniform_keys
from paper_2309_04581_b200.scene import Camera, EmitterSet, make_scene
from paper_2309_04581_b200.surface import Dielectric, Lambertian, Mirror, TriangleMesh

pytestmark = pytest.mark.gpu


def T(a, dev, dtype=None):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev)


# ------------------------------------------------------------------ K1 ---

def test_uniform_bit_exact(cuda, rng):
    keys = np.stack([rng.integers(-2**40, 2**40, 50000), rng.integers(0, 2**31, 50000),
                     rng.integers(0, 64, 50000), rng.integers(0, 8, 50000),
                     rng.integers(0, 9, 50000), rng.integers(0, 1024, 50000)], 1)
    keys[:5] = [[0, 0, 0, 0, 0, 0], [-1, -1, -1, -1, -1, -1], [2**62, 7, 3, 1, 2, 0],
                [7, 5, 3, 1, orng.BSDF_U, 0], [9, 4, 2, 3, orng.BSDF_U, 0]]
    got = uniform_keys(T(keys, cuda, torch.int64)).cpu().numpy()
    want = orng.uniform(*keys.T)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("spp", [1, 2, 4, 16])
def test_primary_rays_bit_exact(cuda, spp):
    cams = [configs.cfg0().camera] + configs.cfg1_cameras(n=5)
    cams.append(Camera(Transform.look_at((0.3, -2, 1.5), (0, 0.2, -1)), math.radians(63), (37, 23)))
    for cam in cams:
        cp = pack_camera(cam)
        w, h = cam.resolution
        pix = np.repeat(np.arange(w * h), spp)[:20000]
        smp = np.tile(np.arange(spp), w * h)[:20000]
        o, d = primary_rays(cam, T(pix, cuda, torch.int64), T(smp, cuda, torch.int64), 11, spp)
        jx, jy = tracer.sample_jitter(11, pix, smp, spp)
        oo, od = tracer.primary_rays(cp, pix, jx, jy)
        assert np.array_equal(o.cpu().numpy(), oo)
        assert np.array_equal(d.cpu().numpy(), od)


# ------------------------------------------------------------------ K2/K3 -

def _random_rays(rng, n, radius=3.0):
    o = rng.normal(size=(n, 3))
    o = radius * o / np.linalg.norm(o, axis=1, keepdims=True)
    target = rng.uniform(-0.6, 0.6, (n, 3))
    d = target - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    inner = rng.uniform(-0.3, 0.3, (n // 4, 3))
    di = rng.normal(size=(n // 4, 3))
    di /= np.linalg.norm(di, axis=1, keepdims=True)
    return np.concatenate([o, inner]), np.concatenate([d, di])


def _soup(rng, n=1000):
    a = rng.uniform(-1, 1, (n, 3))
    tri = a[:, None, :] + rng.normal(0, 0.15, (n, 3, 3))
    return tri


def test_bvh_nearest_bit_exact(cuda, rng):
    scene = configs.cfg1()
    pk = pack_scene(scene)
    r = Renderer(pk)
    o, d = _random_rays(rng, 40000)
    t, f = r.intersect(T(o, cuda), T(d, cuda))
    ts = TriangleSet(pk["v0"], pk["e1"], pk["e2"])
    wt, wf = ts.nearest(o, d)
    assert np.array_equal(f.cpu().numpy(), wf)
    assert np.array_equal(t.cpu().numpy(), wt)
    assert (wf >= 0).mean() > 0.3
    r.close()


def test_bvh_equals_brute_force_on_soup(cuda, rng):
    # reference tests/test_surface.py:101-113 (BVH == brute force on a soup)
    tri = _soup(rng, 1000)
    idx = np.arange(3000).reshape(-1, 3)
    meshes = []
    for k in range(0, 1000, 250):
        sub = tri[k:k + 250].reshape(-1, 3)
        meshes.append(TriangleMesh(sub, np.arange(750).reshape(-1, 3), Lambertian(np.full(3, 0.5))))
    pk = pack_scene(make_scene(meshes=meshes))
    r = Renderer(pk)
    o = rng.uniform(-2, 2, (10000, 3))
    d = rng.normal(size=(10000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, f = r.intersect(T(o, cuda), T(d, cuda))
    ts = TriangleSet(pk["v0"], pk["e1"], pk["e2"])
    bt, bf = ts.brute_nearest(o, d)
    assert np.array_equal(f.cpu().numpy(), bf)
    assert np.array_equal(t.cpu().numpy(), bt)
    del idx
    r.close()


def test_any_hit_bit_exact(cuda, rng):
    scene = configs.cfg1()
    pk = pack_scene(scene)
    r = Renderer(pk)
    o, d = _random_rays(rng, 20000)
    tmin = rng.uniform(0, 1.0, len(o))
    tmax = tmin + rng.uniform(0, 4.0, len(o))
    hit = r.intersect(T(o, cuda), T(d, cuda), T(tmin, cuda), T(tmax, cuda), blocker=True,
                      any_hit=True)
    want = TriangleSet(pk["bv0"], pk["be1"], pk["be2"]).any_hit(o, d, tmin, tmax)
    assert np.array_equal(hit.cpu().numpy(), want)
    r.close()


# ------------------------------------------------------------------ K5/K6 -

def _field_points(rng, fp, n=20000):
    lo, hi = fp["bbox_lo"], fp["bbox_hi"]
    p = rng.uniform(lo, hi, (n, 3))
    # boundaries: the box faces and exact level-cell boundaries
    p[:6] = [lo, hi, [lo[0], hi[1], 0.0], [0.0, 0.0, 0.0], [hi[0], 0.1, lo[2]], [-1e-9, 1e-9, 0.5]]
    k = rng.integers(0, 16, 200)
    p[6:206, 0] = lo[0] + k * (hi[0] - lo[0]) / 16.0
    return p


@pytest.mark.parametrize("cfg", [0, 1, 4])
def test_encode_bit_exact(cuda, rng, cfg):
    field = configs.network(cfg)
    scene = make_scene(field=field)
    r = Renderer(scene)
    fp = r.pack["field"]
    p = _field_points(rng, fp)
    feat, idx = r.field_encode(T(p, cuda))
    wfeat, widx = neural_encode(fp, p, want_index=True)
    assert np.array_equal(idx.cpu().numpy().astype(np.uint32), widx)
    assert np.array_equal(feat.cpu().numpy(), wfeat)
    r.close()


@pytest.mark.parametrize("cfg", [0, 1, 4])
def test_field_sample_matches_oracle(cuda, rng, cfg):
    field = configs.network(cfg)
    r = Renderer(make_scene(field=field))
    fp = r.pack["field"]
    p = _field_points(rng, fp, 8192 + 77)
    d = rng.normal(size=p.shape)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    sigma, rgb, ev = r.field_sample(T(p, cuda), T(d, cuda))
    ws, wrgb = neural_mlp(fp, neural_encode(fp, p), d)
    sigma = sigma.cpu().numpy().astype(np.float64)
    rgb = rgb.cpu().numpy().astype(np.float64)
    assert ev.cpu().numpy().all()
    assert np.abs(sigma / ws - 1).max() < 2e-3
    assert np.abs(rgb - wrgb).max() < 2e-3 * max(1.0, np.abs(wrgb).max())
    # most samples agree to float32 accumulation-order level
    assert np.median(np.abs(sigma / ws - 1)) < 1e-5
    r.close()


@pytest.mark.parametrize("cfg", [0, 1])
def test_occupancy_bits_bit_exact(cuda, cfg):
    field = configs.network(cfg)
    r = Renderer(make_scene(field=field))
    got = r.occupancy()
    want = build_occupancy(r.pack["field"])
    assert np.array_equal(got, want)
    r.close()


# ------------------------------------------------------------- frames ----

def _crop(w, h, size, cx=None, cy=None):
    cx = w // 2 if cx is None else cx
    cy = h // 2 if cy is None else cy
    ys, xs = np.meshgrid(np.arange(cy - size // 2, cy + size // 2),
                         np.arange(cx - size // 2, cx + size // 2), indexing="ij")
    return (ys * w + xs).reshape(-1).astype(np.int64)


def test_cfg0_full_frame_parity(cuda):
    scene = configs.cfg0()
    r = Renderer(scene)
    out = r.render_pixels(scene.camera, 1, 0).cpu().numpy().reshape(64, 64, 3)
    stats = dict(r.last_stats)
    st = {}
    want = tracer.render(r.pack, pack_camera(scene.camera), 1, 0, stats=st)
    assert np.abs(out - want).max() < 1e-3
    assert np.abs(out - want).mean() < 1e-5
    assert stats["nerf_samples"] == st["nerf_samples"]
    r.close()


def test_cfg1_crop_parity(cuda):
    scene = configs.cfg1()
    r = Renderer(scene)
    pix = _crop(800, 800, 48)
    out = r.render_pixels(scene.camera, 1, 0, pixels=T(pix.astype(np.int32), cuda)).cpu().numpy()
    st = {}
    want = tracer.render(r.pack, pack_camera(scene.camera), 1, 0, pixels=pix, stats=st)
    assert np.abs(out - want).max() < 1e-3
    assert r.last_stats["nerf_samples"] == st["nerf_samples"]
    r.close()


def _sparse_field(seed=5, frac=0.35):
    field = configs.network(0)
    g = field.occupancy_res
    rng = np.random.default_rng(seed)
    cells = rng.random(g ** 3) < frac
    words = np.zeros((g ** 3 + 31) // 32, np.uint32)
    idx = np.nonzero(cells)[0]
    np.bitwise_or.at(words, idx >> 5, (np.uint32(1) << (idx & 31).astype(np.uint32)))
    field.occupancy_bits = words
    return field


def test_sparse_occupancy_dda_parity(cuda):
    """Injected 35 %-occupied bitfield (the random-init fog is all
    occupied, so skipping must be tested on a sparse grid): the DDA must
    evaluate exactly the oracle's sample set, in order."""
    scene = configs.cfg0(field=_sparse_field())
    r = Renderer(scene)
    pix = _crop(64, 64, 32)
    cap = 2_000_000
    rec = torch.zeros((cap, 4), dtype=torch.int32, device=cuda)
    r.set_trace(rec, cap)
    out = r.render_pixels(scene.camera, 1, 0, pixels=T(pix.astype(np.int32), cuda)).cpu().numpy()
    n_rec = r.last_stats["trace_records"]
    got = rec[:n_rec].cpu().numpy().astype(np.int64)
    trace = []
    st = {}
    want_img = tracer.render(r.pack, pack_camera(scene.camera), 1, 0, pixels=pix, stats=st,
                             trace=trace)
    want = np.concatenate([np.stack(t, 1) for t in trace]).astype(np.int64)
    key = lambda a: a[np.lexsort((a[:, 2], a[:, 1], a[:, 0]))]
    assert np.array_equal(key(got), key(want))
    assert np.abs(out - want_img).max() < 1e-3
    r.close()


# ------------------------------------------------ dense-grid field plugin --

def _dense_field(seed=0):
    rng = np.random.default_rng(seed)
    return RadianceGrid((-1.5,) * 3, (1.5,) * 3, rng.uniform(0.5, 1.5, (8, 9, 10)),
                        rng.uniform(0, 1, (8, 9, 10, 3)))


def _dense_scenes():
    v, f = assets.icosphere(0.4, 2)
    cam = Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(40), (32, 32))
    yield "mirror", make_scene(field=_dense_field(), meshes=[TriangleMesh(v, f, Mirror(np.full(3, 0.9)))],
                               camera=cam, spp=1, n_bounces=2, march_step=3 * math.sqrt(3) / 256), 1
    yield "glass", make_scene(field=_dense_field(1), meshes=[TriangleMesh(v, f, Dielectric(1.5))],
                              camera=cam, spp=1, n_bounces=4, march_step=3 * math.sqrt(3) / 256), 1
    bv, bf = assets.box((-2, -2, -2), (2, 2, 2), inward=True)
    qv, qf = assets.quad((-1, -1, -1.9), (2, 0, 0), (0, 2, 0))
    room = [TriangleMesh(bv, bf, Lambertian(np.full(3, 0.6))),
            TriangleMesh(qv, qf, Lambertian(np.zeros(3)), emission=np.array((3.0, 2.0, 1.0)))]
    cam2 = Camera(Transform.look_at([0, 0, 1.5], [0, 0, -1]), math.radians(60), (24, 24))
    yield "room", make_scene(field=RadianceGrid.constant((-2,) * 3, (2,) * 3, 0.3, (0.2, 0.1, 0.0)),
                             meshes=room, camera=cam2, spp=4, seed=5, n_bounces=6), 4
    sv, sf = assets.quad((-4, -4, 3.0), (8, 0, 0), (0, 8, 0))
    em = EmitterSet([[[-1, -1, 6], [1, -1, 6], [0, 1, 6]]], [0.7])
    cam3 = Camera(Transform.look_at([0, 0, -3], [0, 0, 0]), math.radians(25), (8, 8))
    yield "shadow", make_scene(field=RadianceGrid.constant((-1,) * 3, (1,) * 3, 1.0, (1, 1, 1)),
                               meshes=[TriangleMesh(sv, sf, Lambertian(np.full(3, 0.5)))],
                               emitters=em, camera=cam3, march_step=0.02, spp=4, seed=9), 4


@pytest.mark.parametrize("name", ["mirror", "glass", "room", "shadow"])
def test_dense_grid_scenes_match_oracle(cuda, name):
    scene, spp = {n: (s, k) for n, s, k in _dense_scenes()}[name]
    r = Renderer(scene)
    w, h = scene.camera.resolution
    out = r.render_pixels(scene.camera, spp, scene.render.seed).cpu().numpy().reshape(h, w, 3)
    want = tracer.render(r.pack, pack_camera(scene.camera), spp, scene.render.seed)
    assert np.abs(out - want).max() < 1e-9
    assert out.mean() > 0.01
    r.close()


# ------------------------------------------------------- frame edge cases

@pytest.mark.parametrize("res,spp", [((37, 21), 1), ((37, 21), 4), ((1, 1), 3), ((17, 33), 2)])
def test_full_frame_odd_shapes_and_spp(cuda, res, spp):
    """Full frames whose sides are not multiples of the 16x16 slot tiles
    (partial edge tiles of tiled_pixel), stratified (4) and plain (2, 3) spp."""
    field = NeuralField.random(3, n_levels=8, n_features=2, log2_table=12, n_min=16, n_max=128,
                               occupancy_res=32)
    v, f = assets.icosphere(0.4, 2)
    cam = Camera(Transform.look_at((0.4, 0.3, 3), (0, 0, 0)), math.radians(40.0), res)
    scene = make_scene(field=field, meshes=[TriangleMesh(v, f, Dielectric(1.5))], camera=cam,
                       spp=spp, n_bounces=3, march_step=configs.MARCH_STEP, seed=4)
    r = Renderer(scene)
    out = r.render_pixels(cam, spp, 4).cpu().numpy()
    st = {}
    want = tracer.render(r.pack, pack_camera(cam), spp, 4, stats=st).reshape(-1, 3)
    assert out.shape == want.shape
    assert np.abs(out - want).max() < 1e-3
    assert r.last_stats["nerf_samples"] == st["nerf_samples"]
    r.close()


def test_empty_pixel_list(cuda):
    scene = configs.cfg0()
    r = Renderer(scene)
    out = r.render_pixels(scene.camera, 1, 0, pixels=torch.zeros(0, dtype=torch.int32, device=cuda))
    assert out.shape == (0, 3)
    assert r.last_stats["paths"] == 0
    r.close()


@pytest.mark.parametrize("continuous", [True, False])
def test_multi_chunk_frame_equals_single_chunks(cuda, continuous):
    """A call with more paths than one wavefront chunk (2^23 for this F = 2 field) is rendered
    as several chunks back to back (new rays, queues and march rounds per
    chunk); every pixel must come out as when it is rendered in a call of
    its own that fits one chunk (paths are keyed by pixel and sample)."""
    scene = configs.cfg0()
    r = Renderer(scene)
    r.set_march(continuous)
    spp = 2100                                   # 4096 px x 2100 spp = 8.6 M paths: 2 chunks
    w, h = scene.camera.resolution
    full = r.render_pixels(scene.camera, spp, 2).cpu().numpy()
    samples_full = r.last_stats["nerf_samples"]
    assert r.last_stats["paths"] == w * h * spp
    parts, samples = [], 0
    for lo in range(0, w * h, 1024):             # 1024 px x 2100 spp = 2.2 M paths: 1 chunk
        pix = torch.arange(lo, lo + 1024, dtype=torch.int32, device=cuda)
        parts.append(r.render_pixels(scene.camera, spp, 2, pixels=pix).cpu().numpy())
        samples += r.last_stats["nerf_samples"]
    assert np.array_equal(full, np.concatenate(parts))
    assert samples_full == samples
    r.close()
