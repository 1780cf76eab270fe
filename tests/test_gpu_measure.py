"""GPU tests of the measurement hooks bench.py relies on: the per-stage
profiler (hrt_set_profile), the batch statistics, the gather-roofline probe
(hrt_gather_peak), and that profiling / the shadow queue / the device-driven
rounds leave the image bit-identical."""

import numpy as np
import pytest
import torch

from paper_2309_04581_b200 import configs
from paper_2309_04581_b200.renderer import Renderer

pytestmark = pytest.mark.gpu


def _crop(w, size=48):
    ys, xs = np.meshgrid(np.arange(400 - size // 2, 400 + size // 2),
                         np.arange(400 - size // 2, 400 + size // 2), indexing="ij")
    return torch.as_tensor((ys * w + xs).reshape(-1).astype(np.int32), device="cuda")


def test_stage_profile_and_stats():
    scene = configs.cfg1()
    r = Renderer(scene)
    pix = _crop(800)
    plain = r.render_pixels(scene.camera, 1, 0, pixels=pix).clone()
    s0 = dict(r.last_stats)
    assert all(v == 0.0 for v in s0["stage_ms"].values())
    r.set_profile(True)
    prof = r.render_pixels(scene.camera, 1, 0, pixels=pix).clone()
    s1 = dict(r.last_stats)
    r.set_profile(False)
    assert torch.equal(plain, prof)
    st = s1["stage_ms"]
    assert st["field"] > 0 and st["intersect"] > 0 and st["composite"] > 0
    assert sum(st.values()) <= s1["ms"] * 1.05
    assert s1["nerf_samples"] == s0["nerf_samples"] > 0
    assert s1["batch_rows"] >= s1["evaluated"] >= s1["nerf_samples"]
    r.close()


def test_gather_peak_probe():
    r = Renderer(configs.cfg1())
    lsu, tex = r.gather_peak(0), r.gather_peak(1)
    assert 100.0 < lsu < 50000.0 and 100.0 < tex < 50000.0
    r.close()


def test_stats_do_not_overflow_int32():
    """64-bit frame counters: 2^20-path chunks x many samples exceed 2^31."""
    scene = configs.cfg4(res=(512, 512))
    scene.render.spp = 64
    scene.render.n_bounces = 1
    r = Renderer(scene)
    r.render_pixels(scene.camera, 64, 0)
    s = r.last_stats
    assert s["paths"] == 512 * 512 * 64
    assert s["nerf_samples"] > 2 ** 31
    assert s["shadow_rays"] > 2 ** 31
    r.close()


def test_render_host_pinned_and_pageable_agree():
    """hrt_render_host: pinned caller buffers (direct DMA) and pageable ones
    (staged) give the device path's frame bit for bit."""
    scene = configs.cfg0()
    r = Renderer(scene)
    dev = r.render_pixels(scene.camera, 1, 0).cpu().numpy()
    pageable = r.render_host(scene.camera, 1, 0)
    out = Renderer.pinned((64 * 64, 3), np.float64)
    r.render_host(scene.camera, 1, 0, out=out)
    assert np.array_equal(dev, pageable) and np.array_equal(dev, out)
    pix = Renderer.pinned((100,), np.int32)
    pix[:] = np.arange(100, 200)
    sub = r.render_host(scene.camera, 1, 0, pixels=pix)
    assert np.array_equal(sub, dev[100:200])
    r.close()
