"""GPU parity on the features of BASELINE configs 2-4 at test scale:
GPU BVH refit of moving meshes (cfg3), shadow rays from NeRF samples with
an F=4 softplus HDR field and an occluding torus (cfg4), and stochastic
Lambertian bounces lit by the NeRF (cfg2)."""

import math

import numpy as np
import pytest
import torch

from oracle import tracer
from oracle.geometry import TriangleSet
from paper_2309_04581_b200 import assets, configs
from paper_2309_04581_b200.core import Transform
from paper_2309_04581_b200.field import NeuralField
from paper_2309_04581_b200.pack import pack_camera, pack_scene
from paper_2309_04581_b200.renderer import Renderer, renderer_for
from paper_2309_04581_b200.scene import Camera, EmitterSet, RenderConfig, Scene
from paper_2309_04581_b200.surface import Dielectric, Lambertian, Mirror, TriangleMesh

pytestmark = pytest.mark.gpu
STEP = configs.MARCH_STEP


def crop(w, h, size, cx=None, cy=None):
    cx = w // 2 if cx is None else cx
    cy = h // 2 if cy is None else cy
    ys, xs = np.meshgrid(np.arange(cy - size // 2, cy + size // 2),
                         np.arange(cx - size // 2, cx + size // 2), indexing="ij")
    return (ys * w + xs).reshape(-1).astype(np.int64)


def small_field(seed=7, act="sigmoid", F=2):
    return NeuralField.random(seed, n_levels=8, n_features=F, log2_table=13, n_min=16, n_max=256,
                              out_activation=act, occupancy_res=32)


def moving_scene(frame, n=20):
    radii, centres, kinds, vel = configs.cfg3_layout()
    base_v, base_f = assets.icosphere(1.0, 2)
    meshes = []
    for i in range(n):
        bsdf = (Mirror(np.full(3, 0.9)), Dielectric(1.5), Lambertian(np.full(3, 0.7)))[kinds[i]]
        meshes.append(TriangleMesh(base_v * radii[i] * 2 + centres[i] * 0.6 + frame * vel[i] * 8,
                                   base_f, bsdf, name=f"s{i}"))
    cam = Camera(configs.look_at_safe((0.0, 0.4, 4.5)), math.radians(40.0), (96, 64))
    return Scene(camera=cam, render=RenderConfig(spp=1, n_bounces=4, march_step=STEP, seed=0,
                                                 threshold=1e-4, sample_cap=1024, early_t=1e-4),
                 field=small_field(), meshes=meshes)


def test_gpu_refit_equals_rebuild_and_oracle(cuda, rng):
    scene = moving_scene(0)
    r = renderer_for(scene)
    w, h = scene.camera.resolution
    before = r.render_pixels(scene.camera, 1, 0).cpu().numpy()
    # move every sphere, refit in place (same renderer, scene.version bump)
    moved = moving_scene(1)
    for m, m2 in zip(scene.meshes, moved.meshes):
        m.vertices = m2.vertices
        m.recompute_normals()
    scene.touch()
    r2 = renderer_for(scene)
    assert r2 is r                                   # refit, not a new upload
    refit = r.render_pixels(scene.camera, 1, 0).cpu().numpy()
    fresh_r = Renderer(moved)
    fresh = fresh_r.render_pixels(moved.camera, 1, 0).cpu().numpy()
    assert not np.array_equal(before, refit)
    assert np.array_equal(refit, fresh)              # hits do not depend on the tree
    pk = pack_scene(moved)
    o = rng.normal(size=(20000, 3)) * 0.2 + [0.0, 0.4, 4.5]
    d = rng.uniform(-1, 1, (20000, 3)) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, f = r.intersect(torch.as_tensor(o, device=cuda), torch.as_tensor(d, device=cuda))
    wt, wf = TriangleSet(pk["v0"], pk["e1"], pk["e2"]).nearest(o, d)
    assert np.array_equal(f.cpu().numpy(), wf) and np.array_equal(t.cpu().numpy(), wt)
    pix = crop(w, h, 16)
    st = {}
    want = tracer.render(pk, pack_camera(moved.camera), 1, 0, pixels=pix, stats=st)
    got = refit.reshape(-1, 3)[pix]
    assert np.abs(got - want).max() < 1e-3
    fresh_r.close()
    r.close()


def shadow_scene(F=4):
    field = small_field(seed=11, act="softplus", F=F)
    lv, lf = assets.quad((-0.5, 2.0, -0.5), (1.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    light = TriangleMesh(lv, lf, Lambertian(np.zeros(3)), emission=np.full(3, 10.0))
    tv, tf = assets.torus(major=0.55, minor=0.18, nu=40, nv=24, seed=4, amplitude=0.03)
    tv = tv[:, [0, 2, 1]] + np.array([0.0, 1.1, 0.0])
    torus = TriangleMesh(tv, tf[:, ::-1].copy(), Lambertian(np.full(3, 0.5)))
    em = EmitterSet(lv[lf].reshape(-1, 3, 3), [1.0, 1.0])
    cam = Camera(configs.look_at_safe((0.0, 0.3, 4.0)), math.radians(40.0), (64, 48))
    return Scene(camera=cam, render=RenderConfig(spp=4, n_bounces=3, march_step=0.05, seed=3,
                                                 threshold=1e-4, sample_cap=1024, early_t=1e-4),
                 field=field, meshes=[light, torus], emitters=em)


def test_gpu_neural_shadows_hdr(cuda):
    """cfg4 features: F=4 encode, softplus HDR radiance, shadow rays from
    every contributing NeRF sample toward an area light, occluded by a torus."""
    scene = shadow_scene()
    r = Renderer(scene)
    w, h = scene.camera.resolution
    pix = crop(w, h, 16, cx=32, cy=20)
    got = r.render_pixels(scene.camera, 4, 3,
                          pixels=torch.as_tensor(pix.astype(np.int32), device=cuda)).cpu().numpy()
    stats = dict(r.last_stats)
    st = {}
    want = tracer.render(r.pack, pack_camera(scene.camera), 4, 3, pixels=pix, stats=st)
    assert stats["shadow_rays"] > 0
    assert stats["nerf_samples"] == st["nerf_samples"]
    rel = np.abs(got - want) / np.maximum(1.0, np.abs(want))
    assert rel.max() < 1e-3
    assert want.max() > 0.1
    r.close()


def test_shadowed_frame_pipelines_agree_at_scale(cuda):
    """A wide shadowed frame (the shadow scene at 256 x 192 x 8 spp: 393k
    paths, batches of millions of rows, thousands of warps per round): the
    device-driven march - shadow rays set up when the samples are generated,
    their codes double-buffered against the previous batch's composite -
    equals the unfused trace-mode pipeline (generate -> field -> shadow
    set-up -> trace -> composite, one kernel each) bit for bit, in the
    continuous and in the bounce-by-bounce march, with equal sample and
    shadow-ray counts."""
    scene = shadow_scene()
    scene.camera = Camera(configs.look_at_safe((0.0, 0.3, 4.0)), math.radians(40.0), (256, 192))
    imgs, stats = [], []
    for mode in ("continuous", "bounce", "unfused"):
        r = Renderer(scene)
        if mode == "bounce":
            r.set_march(False)
        if mode == "unfused":
            rec = torch.zeros((16, 4), dtype=torch.int32, device=cuda)
            r.set_trace(rec, 16)
        imgs.append(r.render_pixels(scene.camera, 8, 3).cpu().numpy())
        stats.append(dict(r.last_stats))
        r.close()
    assert stats[0]["shadow_rays"] > 1_000_000
    for img, st in zip(imgs[1:], stats[1:]):
        assert np.array_equal(imgs[0], img)
        assert st["nerf_samples"] == stats[0]["nerf_samples"]
        assert st["shadow_rays"] == stats[0]["shadow_rays"]


def _render_entry(scene, on, spp, pixels=None):
    """Render with the shadow entry table on or off (HRT_SHADOW_ENTRY is read at create)."""
    import os
    old = os.environ.get("HRT_SHADOW_ENTRY")
    os.environ["HRT_SHADOW_ENTRY"] = "1" if on else "0"
    try:
        r = Renderer(scene)
    finally:
        if old is None:
            del os.environ["HRT_SHADOW_ENTRY"]
        else:
            os.environ["HRT_SHADOW_ENTRY"] = old
    img = r.render_pixels(scene.camera, spp, 3, pixels=pixels).cpu().numpy()
    st = dict(r.last_stats)
    r.close()
    return img, st


@pytest.mark.parametrize("moved", [False, True])
def test_shadow_entry_table_exact(cuda, moved):
    """Shadow rays started from the light-space entry table (the blocker-tree
    node under which everything a ray from that field cell to that light
    patch can hit lies, or no traversal at all) decide exactly what
    traversals from the root decide: bit-identical images and equal sample
    and shadow-ray counts, with the field box in place and moved (rotated +
    shifted, so the table's grid covers a transformed box)."""
    scene = shadow_scene()
    scene.camera = Camera(configs.look_at_safe((0.0, 0.3, 4.0)), math.radians(40.0), (160, 120))
    if moved:
        scene.field.world_from_field = Transform.translate((0.15, -0.1, 0.05)).compose(
            Transform.rotate((0.3, 1.0, 0.2), 0.4))
    on, st_on = _render_entry(scene, True, 8)
    off, st_off = _render_entry(scene, False, 8)
    assert st_on["shadow_rays"] > 100_000
    assert st_on["nerf_samples"] == st_off["nerf_samples"]
    assert st_on["shadow_rays"] == st_off["shadow_rays"]
    assert np.array_equal(on, off)


def test_shadow_entry_table_exact_cfg4_geometry(cuda):
    """The same on the full cfg4 blockers (300k-triangle displaced torus,
    deep tree) with a small field: a 48 x 48 x 16 spp crop under the torus."""
    scene = configs.cfg4(field=small_field(seed=11, act="softplus", F=4), res=(480, 270))
    w, h = scene.camera.resolution
    pix = torch.as_tensor(crop(w, h, 48, cx=240, cy=120).astype(np.int32), device=cuda)
    on, st_on = _render_entry(scene, True, 16, pix)
    off, st_off = _render_entry(scene, False, 16, pix)
    assert st_on["shadow_rays"] > 100_000
    assert st_on["shadow_rays"] == st_off["shadow_rays"]
    assert np.array_equal(on, off)


def test_gpu_cfg2_lambertian_crop(cuda):
    """cfg2: diffuse plane + 50k-triangle blob lit only by the NeRF, 16 spp
    stratified. The GPU reuses the reference RNG streams, so paths match the
    oracle except where cos/sin last-ulp differences move a hit."""
    scene = configs.cfg2()
    r = Renderer(scene)
    w, h = scene.camera.resolution
    pix = crop(w, h, 8, cx=256, cy=300)
    got = r.render_pixels(scene.camera, 16, 0,
                          pixels=torch.as_tensor(pix.astype(np.int32), device=cuda)).cpu().numpy()
    want = tracer.render(r.pack, pack_camera(scene.camera), 16, 0, pixels=pix)
    d = np.abs(got - want)
    assert np.mean(d < 1e-4) > 0.95
    assert d.mean() < 1e-3
    r.close()


def test_gpu_rigid_refit_equals_host_moved_scene():
    """hrt_refit_rigid (transforms only, faces/normals/trees rebuilt on the GPU)
    renders bit-identically to a renderer built from host-moved meshes."""
    radii, centres, kinds, vel = configs.cfg3_layout()
    n = 24
    layout = (radii[:n] * 2, centres[:n] * 0.6, kinds[:n], vel[:n] * 8)
    base_v, base_f = assets.icosphere(1.0, 2)

    def scene_at(frame, spawn_eps=None):
        xf = configs.cfg3_transforms(frame, layout)
        meshes = [TriangleMesh(configs.apply_rigid(base_v, xf[i]), base_f,
                               (Mirror(np.full(3, 0.9)), Dielectric(1.5), Lambertian(np.full(3, 0.7)))[kinds[i]])
                  for i in range(n)]
        cam = Camera(configs.look_at_safe((0.0, 0.4, 4.5)), math.radians(40.0), (80, 48))
        return Scene(camera=cam, render=RenderConfig(spp=2, n_bounces=4, march_step=STEP, seed=0,
                                                     threshold=1e-4, sample_cap=1024, early_t=1e-4),
                     field=small_field(), meshes=meshes, spawn_eps=spawn_eps)

    s0 = scene_at(0)
    r = Renderer(s0)
    r.set_rigid_base([base_v] * n, [base_f] * n)
    for frame in (3, 11):
        r.refit_rigid(configs.cfg3_transforms(frame, layout))
        got = r.render_pixels(s0.camera, 2, 0).clone()
        st = dict(r.last_stats)
        sf = scene_at(frame, spawn_eps=s0.spawn_eps)
        ref = Renderer(sf)
        want = ref.render_pixels(sf.camera, 2, 0)
        assert torch.equal(got, want), float((got - want).abs().max())
        assert st["nerf_samples"] == ref.last_stats["nerf_samples"]
        ref.close()
    r.close()


@pytest.mark.parametrize("which", ["cfg1", "cfg1_full", "shadows", "cfg2", "moving"])
def test_gpu_continuous_march_equals_bounce_loop(cuda, which):
    """The continuous wavefront march (paths advance to their next bounce
    inside the march rounds, kern::advance) against the reference's
    bounce-by-bounce loop (render.py:214) on the same renderer: images, NeRF
    sample counts, shadow rays and bounce rays are identical, bit for bit."""
    if which == "cfg1":
        scene, spp, size, cx, cy = configs.cfg1(), 1, 48, 400, 400
    elif which == "cfg1_full":          # 640 k paths: wide rounds first, 8-lane tail rounds last
        scene, spp, size, cx, cy = configs.cfg1(), 1, None, None, None
    elif which == "shadows":
        scene, spp, size, cx, cy = shadow_scene(), 4, 16, 32, 20
    elif which == "cfg2":
        scene, spp, size, cx, cy = configs.cfg2(), 4, 16, 256, 300
    else:
        scene, spp, size, cx, cy = moving_scene(3), 2, 32, 48, 32
    r = Renderer(scene)
    w, h = scene.camera.resolution
    pix = None if size is None else torch.as_tensor(crop(w, h, size, cx=cx, cy=cy).astype(np.int32),
                                                     device=cuda)
    out = {}
    for continuous in (True, False):
        r.set_march(continuous)
        img = r.render_pixels(scene.camera, spp, 5, pixels=pix).cpu().numpy()
        out[continuous] = (img, dict(r.last_stats))
    (a, sa), (b, sb) = out[True], out[False]
    assert np.array_equal(a, b)
    # ("evaluated" counts field-engine rows incl. samples generated past an
    # early-out inside a batch; it depends on the round sizes, not a result)
    for key in ("nerf_samples", "shadow_rays", "bounce_rays"):
        assert sa[key] == sb[key], key
    assert sa["rounds"] <= sb["rounds"]
    r.close()


@pytest.mark.parametrize("n_bounces,threshold,sample_cap,early_t", [
    (0, 1e-4, 1024, 1e-4),       # march only, no surface interaction
    (1, 1e-4, 1024, 1e-4),
    (6, 1e-4, 1024, 1e-4),       # more bounces than most paths live
    (4, 0.5, 1024, 1e-4),        # throughput threshold kills paths at their first hit
    (4, 1e-4, 1, 1e-4),          # sample cap reached on the first sample: later bounces march nothing
    (4, 1e-4, 37, 1e-4),         # cap in the middle of a round / bounce
    (4, 1e-4, 0, 0.6),           # early-out after a few samples, then shading continues
])
def test_gpu_continuous_march_edge_configs(cuda, n_bounces, threshold, sample_cap, early_t):
    """Continuous march vs the bounce-by-bounce loop on RenderConfig edges
    (hrt_set_config): halted paths (cap / early-out) must still be shaded and
    continue through their remaining bounces with zero samples, exactly as
    the per-bounce loop does."""
    scene = moving_scene(5)
    r = Renderer(scene)
    cfg = (n_bounces, threshold, scene.render.march_step, r.pack["spawn_eps"], sample_cap, early_t)
    r.set_config(cfg)
    w, h = scene.camera.resolution
    pix = torch.as_tensor(crop(w, h, 32, cx=48, cy=32).astype(np.int32), device=cuda)
    out = {}
    for continuous in (True, False):
        r.set_march(continuous)
        img = r.render_pixels(scene.camera, 2, 9, pixels=pix).cpu().numpy()
        out[continuous] = (img, dict(r.last_stats))
    (a, sa), (b, sb) = out[True], out[False]
    assert np.array_equal(a, b)
    for key in ("nerf_samples", "bounce_rays"):
        assert sa[key] == sb[key], key
    if sample_cap == 1:
        assert sa["nerf_samples"] <= 2 * pix.numel()
    r.close()


@pytest.mark.parametrize("sample_cap,early_t,threshold", [
    (1, 1e-4, 1e-4),             # cap reached on the first sample of the path
    (37, 1e-4, 1e-4),            # cap inside a round and inside a bounce
    (0, 0.6, 1e-4),              # in-march early-out after a few samples, shading continues
    (1024, 1e-4, 0.5),           # post-bounce throughput threshold kills paths at the first hit
])
def test_gpu_march_limits_vs_oracle(cuda, sample_cap, early_t, threshold):
    """SURVEY P5 limits (1024-sample cap, in-march early-out) against the
    ORACLE's own implementation of them (oracle/tracer.py march), not only
    against the GPU's bounce loop: images within 1e-3, NeRF sample counts
    equal."""
    scene = moving_scene(5)
    scene.render.sample_cap, scene.render.early_t, scene.render.threshold = sample_cap, early_t, threshold
    r = Renderer(scene)
    assert (r.pack["sample_cap"], r.pack["early_t"], r.pack["threshold"]) == (sample_cap, early_t, threshold)
    w, h = scene.camera.resolution
    pix = crop(w, h, 16, cx=48, cy=32)
    got = r.render_pixels(scene.camera, 2, 9,
                          pixels=torch.as_tensor(pix.astype(np.int32), device=cuda)).cpu().numpy()
    stats = dict(r.last_stats)
    st = {}
    want = tracer.render(r.pack, pack_camera(scene.camera), 2, 9, pixels=pix, stats=st)
    assert stats["nerf_samples"] == st["nerf_samples"]
    assert np.abs(got - want).max() < 1e-3
    if sample_cap == 1:
        assert st["nerf_samples"] <= 2 * len(pix)
    assert want.max() > 0.01
    r.close()
