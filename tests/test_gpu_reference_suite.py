"""The reference's known-answer render tests (reference
pkg/tests/test_render.py) restated against the GPU path through
this package's public API (`trace_path`, `render`, `render_surface_only`,
`render_volume_only`). Closed forms and degeneracy equivalences are the
reference's only reference-pinned parity for the render loop."""

import math

import numpy as np
import pytest

from paper_2309_04581_b200 import (EmitterSet, Lambertian, Mirror, PathRng, RadianceGrid,
                                   Transform, TriangleMesh, make_scene, render, render_surface_only,
                                   render_volume_only, trace_path)
from paper_2309_04581_b200 import assets
from paper_2309_04581_b200.core import Ray
from paper_2309_04581_b200.scene import Camera

pytestmark = pytest.mark.gpu


def emissive_quad(emission=(2.0, 2.0, 2.0), z=0.0, half=4.0):
    v, f = assets.quad((-half, -half, z), (2 * half, 0, 0), (0, 2 * half, 0))
    return TriangleMesh(v, f, Lambertian(np.zeros(3)), emission=np.array(emission))


def test_vacuum_emitter_direct(cuda):                       # test_render.py:47-50
    scene = make_scene(meshes=[emissive_quad()])
    L = trace_path(Ray([0, 0, 3], [0, 0, -1]), scene, PathRng(1))
    assert np.array_equal(L, [2.0, 2.0, 2.0])


def test_homogeneous_slab(cuda):                            # test_render.py:53-57
    field = RadianceGrid.constant((0, 0, 0), (1, 1, 1), 1.0, (1, 1, 1))
    scene = make_scene(field=field, march_step=1e-3)
    L = trace_path(Ray([0.5, 0.5, -1.0], [0, 0, 1]), scene, PathRng(1))
    assert np.allclose(L, 1.0 - math.exp(-1.0), rtol=1e-2)


def test_mirror_behind_slab_two_segment_form(cuda):         # test_render.py:60-72
    rho, r_val = 0.8, 0.6
    field = RadianceGrid.constant((0, 0, 0), (1, 1, 1), 1.0, (r_val, r_val, r_val))
    v, f = assets.quad((-2, -2, 1.0), (4, 0, 0), (0, 4, 0))
    scene = make_scene(field=field, meshes=[TriangleMesh(v, f, Mirror(np.full(3, rho)))],
                       march_step=1e-3)
    L = trace_path(Ray([0.5, 0.5, -1.0], [0, 0, 1]), scene, PathRng(1))
    seg = r_val * (1.0 - math.exp(-1.0))
    assert np.allclose(L, seg + math.exp(-1.0) * rho * seg, rtol=2e-2)


def test_bounce_limit_between_mirrors(cuda):                 # test_render.py:75-83
    v1, f1 = assets.quad((-2, -2, 0.0), (4, 0, 0), (0, 4, 0))
    v2, f2 = assets.quad((-2, -2, 2.0), (0, 4, 0), (4, 0, 0))
    scene = make_scene(meshes=[TriangleMesh(v1, f1, Mirror(np.ones(3))),
                               TriangleMesh(v2, f2, Mirror(np.ones(3)))], n_bounces=5)
    L = trace_path(Ray([0, 0, 1.0], [0, 0, -1]), scene, PathRng(1))
    assert np.array_equal(L, np.zeros(3))


def test_throughput_threshold_terminates(cuda):             # test_render.py:86-90
    field = RadianceGrid.constant((0, 0, 0), (1, 1, 1), 40.0, (1, 1, 1))
    scene = make_scene(field=field, march_step=1e-2, threshold=1e-3)
    L = trace_path(Ray([0.5, 0.5, -1.0], [0, 0, 1]), scene, PathRng(1))
    assert np.allclose(L, 1.0, rtol=1e-2)


def shadow_scene(r_src):                                    # test_render.py:120-131
    field = RadianceGrid.constant((-1, -1, -1), (1, 1, 1), 1.0, (1, 1, 1))
    v, f = assets.quad((-4, -4, 3.0), (8, 0, 0), (0, 8, 0))
    em = None if r_src is None else EmitterSet([[[-1, -1, 6], [1, -1, 6], [0, 1, 6]]], [r_src])
    cam = Camera(Transform.look_at([0, 0, -3], [0, 0, 0]), math.radians(25), (8, 8))
    return make_scene(field=field, meshes=[TriangleMesh(v, f, Lambertian(np.full(3, 0.5)))],
                      emitters=em, camera=cam, march_step=0.02, spp=4, seed=9)


def test_blocked_contribution_scales_by_one_minus_rsrc(cuda):   # test_render.py:138-141
    blocked = render(shadow_scene(0.7)).pixels
    open_ = render(shadow_scene(0.0)).pixels
    assert np.allclose(blocked, 0.3 * open_, rtol=1e-12)


def test_rsrc_zero_bit_equals_shadow_free(cuda):            # test_render.py:144-147
    assert np.array_equal(render(shadow_scene(0.0)).pixels, render(shadow_scene(None)).pixels)


def room_scene(sigma):                                      # test_render.py:153-162
    field = (RadianceGrid.constant((-2, -2, -2), (2, 2, 2), sigma, (0.0, 0.0, 0.0))
             if sigma is not None else None)
    v, f = assets.box((-2, -2, -2), (2, 2, 2), inward=True)
    room = TriangleMesh(v, f, Lambertian(np.full(3, 0.6)))
    cam = Camera(Transform.look_at([0, 0, 1.5], [0, 0, -1]), math.radians(60), (64, 64))
    return make_scene(field=field, meshes=[room, emissive_quad((3.0, 2.0, 1.0), z=-1.9, half=1.0)],
                      camera=cam, spp=16, seed=5, n_bounces=6)


def test_degeneracy_a_zero_sigma_equals_surface_tracer(cuda):   # test_render.py:165-169
    hybrid = render(room_scene(0.0)).pixels
    surface = render_surface_only(room_scene(None)).pixels
    assert np.array_equal(hybrid, surface)
    assert hybrid.mean() > 0.01


def test_degeneracy_b_mesh_free_equals_volume_tracer(cuda):     # test_render.py:172-178
    rng = np.random.default_rng(3)
    field = RadianceGrid((-1, -1, -1), (1, 1, 1), rng.uniform(0, 2, (6, 6, 6)),
                         rng.uniform(0, 1, (6, 6, 6, 3)))
    cam = Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(40), (32, 32))
    scene = make_scene(field=field, camera=cam, spp=16, seed=3, march_step=0.02)
    hybrid = render(scene).pixels
    volume = render_volume_only(scene).pixels
    assert np.array_equal(hybrid, volume)
    assert hybrid.mean() > 0.05


def test_single_pixel_emitter_exact_at_any_spp(cuda):       # test_render.py:184-190
    cam = Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(20), (1, 1))
    scene = make_scene(meshes=[emissive_quad()], camera=cam)
    for spp in (1, 2, 7):
        assert np.array_equal(render(scene, spp=spp, seed=1).pixels[0, 0], [2.0, 2.0, 2.0])


def test_determinism_and_seed_sensitivity(cuda):            # test_render.py:193-214
    scene = room_scene(0.2)
    a = render(scene, spp=2, seed=11).pixels
    b = render(scene, spp=2, seed=11, threads=4).pixels
    c = render(scene, spp=2, seed=12).pixels
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)


def test_rejects_bad_spp(cuda):                             # test_render.py:217-221
    with pytest.raises(ValueError):
        render(room_scene(0.2), spp=0)
