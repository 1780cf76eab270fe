"""Stochastic parity (BASELINE cfg2: "compared statistically against a
1024-spp reference mean"; north star: "stochastic images agree within Monte
Carlo error at matched spp") and the reference's furnace known-answer test.

Patterns follow the reference's statistical tests: the furnace at 16 spp
within 5 % (`tests/test_render.py:266-272`) and the chi-square goodness of
fit of `tests/test_surface.py:234-251`, applied here to per-pixel z-scores
of GPU estimates against the oracle's 1024-spp mean, with the Monte Carlo
standard error measured from independent GPU seeds.
"""

import math

import numpy as np
import pytest
import torch
from scipy import stats as sst

from oracle import tracer
from paper_2309_04581_b200 import Lambertian, RadianceGrid, TriangleMesh, assets, configs, make_scene, render
from paper_2309_04581_b200.core import Transform
from paper_2309_04581_b200.pack import pack_camera
from paper_2309_04581_b200.renderer import Renderer, primary_rays
from paper_2309_04581_b200.scene import Camera
import oracle_pool

pytestmark = pytest.mark.gpu

SEEDS = 64            # independent 16-spp GPU estimates per pixel (MC error + 1024-spp GPU mean)


def crop(w, h, size, cx, cy):
    ys, xs = np.meshgrid(np.arange(cy - size // 2, cy + size // 2),
                         np.arange(cx - size // 2, cx + size // 2), indexing="ij")
    return (ys * w + xs).reshape(-1).astype(np.int64)


@pytest.fixture(scope="module")
def cfg2_stats(cuda):
    scene = configs.cfg2()
    r = Renderer(scene)
    w, h = scene.camera.resolution
    pix = crop(w, h, 8, cx=256, cy=300)
    pt = torch.as_tensor(pix.astype(np.int32), device=cuda)
    est = np.stack([r.render_pixels(scene.camera, 16, 1000 + k, pixels=pt).cpu().numpy()
                    for k in range(SEEDS)])                          # (SEEDS, px, 3), 16 spp each
    g1024_same = r.render_pixels(scene.camera, 1024, 7, pixels=pt).cpu().numpy()
    want, st = oracle_pool.render(tracer.OracleScene(r.pack), pack_camera(scene.camera), 1024, 7, pix)
    yield {"scene": scene, "r": r, "pix": pix, "est": est, "g1024_same": g1024_same, "oracle1024": want}
    r.close()


def _z(a, b, var):
    lum_a, lum_b = a.mean(axis=-1), b.mean(axis=-1)
    return (lum_a - lum_b) / np.sqrt(var)


def test_cfg2_16spp_within_mc_error_of_oracle_1024spp(cfg2_stats):
    """Each 16-spp GPU estimate (one seed) against the oracle's 1024-spp
    mean (seed 7): per-pixel z-scores with the MC standard error of a
    16-spp estimate measured over 64 GPU seeds; chi-square over the crop
    within the central 99.8 % of chi2(64)."""
    est, want = cfg2_stats["est"], cfg2_stats["oracle1024"]
    lum = est.mean(axis=-1)                                          # (SEEDS, px)
    var16 = lum.var(axis=0, ddof=1)
    assert (var16 > 0).all()
    var = var16 * (1.0 + 1.0 / 16.0)                  # + the oracle mean's own error (<= var16 / 64 x 4)
    n = len(cfg2_stats["pix"])
    lo, hi = sst.chi2.ppf(0.001, n), sst.chi2.ppf(0.999, n)
    failures = 0
    for k in range(4):                                               # four independent estimates
        z = _z(est[k], want, var)
        chi2 = float((z * z).sum())
        failures += not (lo < chi2 < hi)
        assert np.abs(z).max() < 5.0, (k, np.abs(z).max())
    assert failures <= 1


def test_cfg2_gpu_1024spp_mean_vs_oracle_1024spp(cfg2_stats):
    """The GPU's 1024-spp mean (64 seeds x 16 spp) against the oracle's
    1024-spp mean (different streams): z-test at the standard error of the
    difference of the two means, chi-square over the crop."""
    est, want = cfg2_stats["est"], cfg2_stats["oracle1024"]
    lum = est.mean(axis=-1)
    mean = lum.mean(axis=0)
    var_mean = lum.var(axis=0, ddof=1) / SEEDS
    z = (mean - want.mean(axis=-1)) / np.sqrt(2.0 * var_mean)        # both means ~ var16 / 64
    n = len(z)
    assert np.abs(z).max() < 5.0
    assert float((z * z).sum()) < sst.chi2.ppf(0.999, n)
    assert abs(float(z.mean())) < 4.0 / math.sqrt(n)                # no bias


def test_cfg2_matched_spp_shared_streams(cfg2_stats):
    """Same seed, same spp (1024): GPU and oracle consume the same counter
    RNG streams, so the images agree per pixel far inside the 1e-3 bar; a
    path whose Lambertian direction differs by a last-ulp cos/sin
    (surface.py:89-90, libm vs CUDA) moves a pixel by at most its 1/1024
    share."""
    got, want = cfg2_stats["g1024_same"], cfg2_stats["oracle1024"]
    d = np.abs(got - want)
    assert d.max() < 1e-3, d.max()
    assert np.median(d) < 1e-6          # (the fp16-operand MLP alone moves a pixel by ~1e-8)


def test_cfg2_paths_exact_except_listed_near_ties(cuda):
    """Per-path radiance of the cfg2 crop (1024 camera paths, 16 spp):
    every path equals the oracle's to 1e-5 (the fp16-operand MLP's own
    deviation; the median path is ~1e-8 off) except an explicitly listed
    handful (< 1 %) whose diffuse bounce direction differs in the last ulp
    of cos/sin; those are reported by (pixel, sample)."""
    scene = configs.cfg2()
    r = Renderer(scene)
    w, h = scene.camera.resolution
    pix = np.repeat(crop(w, h, 8, cx=256, cy=300), 16)
    smp = np.tile(np.arange(16), len(pix) // 16)
    pt, st = torch.as_tensor(pix, device=cuda), torch.as_tensor(smp, device=cuda)
    o, d = primary_rays(scene.camera, pt, st, 0, 16)
    L = r.trace(o, d, pt, st, 0).cpu().numpy()
    sc = tracer.OracleScene(r.pack)
    oracle_pool.occupancy(sc.field)
    want = tracer.trace_paths(sc, o.cpu().numpy(), d.cpu().numpy(), pix, smp, 0)
    diff = np.abs(L - want).max(axis=1)
    odd = np.nonzero(diff > 1e-5)[0]
    listed = [(int(pix[i]), int(smp[i]), float(diff[i])) for i in odd]
    assert len(odd) <= len(pix) // 100, listed
    assert np.median(diff) < 1e-7
    r.close()


def furnace_scene(res=(64, 64)):
    """The reference furnace preset (assets.py:258-275, restated): a
    uniform emissive medium (sigma 2, radiance 0.8) around an albedo-1
    Lambertian icosphere; energy conservation makes every pixel 0.8."""
    field = RadianceGrid.constant((-2, -2, -2), (2, 2, 2), 2.0, (0.8, 0.8, 0.8))
    v, f = assets.icosphere(0.5, 2)
    sphere = TriangleMesh(v, f, Lambertian(np.ones(3)))
    cam = Camera(Transform.look_at((0.0, 0.0, 1.6), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0)), math.radians(45.0), res)
    return make_scene(field=field, meshes=[sphere], camera=cam, spp=64, n_bounces=8, march_step=0.2, seed=7)


def test_furnace_small_scale(cuda):                                 # test_render.py:266-272
    img = render(furnace_scene(), spp=16, seed=7)
    center = img.pixels[28:36, 28:36].mean()
    assert abs(center - 0.8) / 0.8 < 0.05


def test_furnace_1024spp_converges(cuda):
    """Same preset at 1024 spp: the centre converges to 0.8 within 1 %
    (the reference's acceptance furnace, SPEC "furnace 1024 spp")."""
    scene = furnace_scene((32, 32))
    img = render(scene, spp=1024, seed=3)
    center = img.pixels[12:20, 12:20].mean()
    assert abs(center - 0.8) / 0.8 < 0.01, center
    # and per pixel against the oracle on the same streams
    from paper_2309_04581_b200.pack import pack_scene
    ys, xs = np.meshgrid(np.arange(12, 20), np.arange(12, 20), indexing="ij")
    pix = (ys * 32 + xs).reshape(-1)
    want, _ = oracle_pool.render(tracer.OracleScene(pack_scene(scene)), pack_camera(scene.camera), 1024, 3, pix)
    assert np.abs(img.pixels.reshape(-1, 3)[pix] - want).max() < 1e-3
