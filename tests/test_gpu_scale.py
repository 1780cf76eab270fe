"""Parity at BASELINE's full scale (VERDICT r1 "no parity at cfg3 / cfg4
scale"): the real 1,024,000-triangle, 200-mesh cfg3 forest (frame 0 and
after `hrt_refit_rigid` to frame 29) and the real cfg4 scene (L16 F4 T2^21
softplus network, 300k-triangle torus blocker, area light with shadow rays),
against the CPU oracle.

Bar (north star): BVH face ids and t bit-exact (reference hit contract
`surface.py:377-503`: nearest t, ties to the smaller face id; any-hit
`surface.py:442-478`); images within 1e-3 max abs (cfg4 HDR: relative to
max(1, |L|)); NeRF sample and shadow-ray counts equal.
"""

import numpy as np
import pytest
import torch

from oracle import tracer
from oracle.geometry import TriangleSet
from paper_2309_04581_b200 import assets, configs
from paper_2309_04581_b200.pack import pack_camera, pack_scene
from paper_2309_04581_b200.renderer import Renderer
import oracle_pool

pytestmark = pytest.mark.gpu


def crop(w, h, size, cx, cy):
    ys, xs = np.meshgrid(np.arange(cy - size // 2, cy + size // 2),
                         np.arange(cx - size // 2, cx + size // 2), indexing="ij")
    return (ys * w + xs).reshape(-1).astype(np.int64)


@pytest.fixture(scope="module")
def cfg3(cuda):
    scene = configs.cfg3()
    r = Renderer(scene)
    base_v, base_f = assets.icosphere(1.0, 4)
    r.set_rigid_base([base_v] * len(scene.meshes), [base_f] * len(scene.meshes))
    yield scene, r
    r.close()


def scene_rays(rng, n, cam_pos):
    """Half camera-like rays (from near the eye toward points of the box),
    half secondary-like rays (from points of the box in random directions)."""
    h = n // 2
    o1 = cam_pos + rng.normal(0.0, 0.05, (h, 3))
    d1 = rng.uniform(-1.5, 1.5, (h, 3)) - o1
    o2 = rng.uniform(-1.5, 1.5, (n - h, 3))
    d2 = rng.normal(size=(n - h, 3))
    o, d = np.concatenate([o1, o2]), np.concatenate([d1, d2])
    return o, d / np.linalg.norm(d, axis=1, keepdims=True)


@pytest.mark.parametrize("frame", [0, 29])
def test_cfg3_forest_hits_bit_exact(cfg3, cuda, frame):
    """20k rays against the full 1.02 M-triangle forest after the GPU rigid
    refit to `frame`: nearest face id and t bit-exact vs the oracle's
    intersector over the host-moved faces; any-hit on the blocker trees too."""
    scene, r = cfg3
    r.refit_rigid(configs.cfg3_transforms(frame))
    pk = pack_scene(configs.cfg3(frame=frame, res=(16, 16)))
    assert len(pk["v0"]) == 1_024_000
    rng = np.random.default_rng(100 + frame)
    o, d = scene_rays(rng, 20000, np.array([0.0, 0.4, 4.5]))
    t, f = r.intersect(torch.as_tensor(o, device=cuda), torch.as_tensor(d, device=cuda))
    ts = TriangleSet(pk["v0"], pk["e1"], pk["e2"])
    wt, wf = ts.nearest(o, d)
    f, t = f.cpu().numpy(), t.cpu().numpy()
    assert (wf >= 0).mean() > 0.2                   # a real share of the rays hit a sphere
    assert np.array_equal(f, wf)
    assert np.array_equal(t, wt)
    tmin = np.full(len(o), 1e-4)
    tmax = rng.uniform(0.05, 4.0, len(o))
    hit = r.intersect(torch.as_tensor(o, device=cuda), torch.as_tensor(d, device=cuda),
                      t_min=torch.as_tensor(tmin, device=cuda), t_max=torch.as_tensor(tmax, device=cuda),
                      blocker=True, any_hit=True).cpu().numpy()
    want = TriangleSet(pk["bv0"], pk["be1"], pk["be2"]).any_hit(o, d, tmin, tmax)
    assert 0.05 < want.mean() < 0.95
    assert np.array_equal(hit, want)


def test_cfg3_crop_vs_oracle_after_refit(cfg3, cuda):
    """A 16x16 x 8 spp crop of the 1080p frame after refitting to motion
    frame 29: within 1e-3 of the oracle with equal NeRF sample counts."""
    scene, r = cfg3
    r.refit_rigid(configs.cfg3_transforms(29))
    w, h = scene.camera.resolution
    pix = crop(w, h, 16, cx=1000, cy=560)
    got = r.render_pixels(scene.camera, 8, 0,
                          pixels=torch.as_tensor(pix.astype(np.int32), device=cuda)).cpu().numpy()
    stats = dict(r.last_stats)
    pk = pack_scene(configs.cfg3(frame=29, res=(16, 16)))
    pk["spawn_eps"] = r.pack["spawn_eps"]            # the renderer's (frame-0 scene diagonal)
    want, st = oracle_pool.render(tracer.OracleScene(pk), pack_camera(scene.camera), 8, 0, pix)
    assert stats["nerf_samples"] == st["nerf_samples"]
    err = np.abs(got - want)
    assert err.max() < 1e-3, (err.max(), np.argwhere(err > 1e-3)[:5])
    assert want.mean() > 0.05


def test_cfg4_crop_vs_oracle():
    """cfg4 at full scale: the L16 F4 T2^21 16->4096 softplus HDR network
    (344 MiB table), 300k-triangle displaced torus blocking an area light of
    radiance 10: two 8x8 x 64 spp crops (stratified 8x8) of the 4K frame
    against the oracle - relative error 1e-3, equal NeRF sample and
    shadow-ray counts."""
    scene = configs.cfg4()
    assert len(scene.meshes[1].indices) == 300_000
    r = Renderer(scene)
    w, h = scene.camera.resolution
    # the frame centre (field + shadows only) and the torus' far side (diffuse
    # torus hits, bounce rays back through the shadowed field)
    pix = np.concatenate([crop(w, h, 8, cx=1920, cy=1000), crop(w, h, 8, cx=2300, cy=400)])
    got = r.render_pixels(scene.camera, 64, 0,
                          pixels=torch.as_tensor(pix.astype(np.int32), device="cuda")).cpu().numpy()
    stats = dict(r.last_stats)
    want, st = oracle_pool.render(tracer.OracleScene(r.pack), pack_camera(scene.camera), 64, 0, pix)
    assert stats["nerf_samples"] == st["nerf_samples"]
    assert stats["shadow_rays"] == st["shadow_rays"] > 0
    rel = np.abs(got - want) / np.maximum(1.0, np.abs(want))
    assert rel.max() < 1e-3, (rel.max(), np.argwhere(rel > 1e-3)[:5])
    assert want.max() > 0.1
    r.close()


@pytest.fixture(scope="module")
def cfg1(cuda):
    scene = configs.cfg1()
    r = Renderer(scene)
    yield scene, r
    r.close()


def test_cfg1_other_cameras_crops(cfg1, cuda):
    """cfg1 beyond camera 0: a 16x16 crop at a seeded position
    of each of eight more of the 100 seeded cameras, against the oracle."""
    scene, r = cfg1
    cams = configs.cfg1_cameras()
    g = np.random.default_rng(21)
    for ci in (7, 19, 33, 42, 58, 71, 86, 99):
        cam = cams[ci]
        cx, cy = (int(v) for v in g.integers(200, 600, 2))
        pix = crop(800, 800, 16, cx=cx, cy=cy)
        got = r.render_pixels(cam, 1, 0, pixels=torch.as_tensor(pix.astype(np.int32), device=cuda)).cpu().numpy()
        stats = dict(r.last_stats)
        want, st = oracle_pool.render(tracer.OracleScene(r.pack), pack_camera(cam), 1, 0, pix)
        assert stats["nerf_samples"] == st["nerf_samples"], ci
        assert np.abs(got - want).max() < 1e-3, ci


def test_cfg1_full_frame(cfg1, cuda):
    """A whole 800x800 cfg1 frame (camera 57; 640,000 paths, ~87 M NeRF
    samples on the oracle) against the oracle: max abs < 1e-3, equal NeRF
    sample counts."""
    scene, r = cfg1
    cam = configs.cfg1_cameras()[57]
    got = r.render_pixels(cam, 1, 0).cpu().numpy()
    stats = dict(r.last_stats)
    want, st = oracle_pool.render(tracer.OracleScene(r.pack), pack_camera(cam), 1, 0, np.arange(800 * 800),
                                  parts=512)
    assert stats["nerf_samples"] == st["nerf_samples"]
    err = np.abs(got - want)
    assert err.max() < 1e-3, (err.max(), np.argwhere(err > 1e-3)[:5])
