"""GPU transport operator (emitter estimation, reference emitters.py:73-166)
vs the reference's own build_transport output (tests/golden/transport.npz),
its validation errors, and the linearity it exists for: A @ emission equals
the surface-only render at the same depth and seeds."""

import math

import numpy as np
import pytest

import golden_scenes as gs
from paper_2309_04581_b200 import renderer
from paper_2309_04581_b200.core import Transform
from paper_2309_04581_b200.field import RadianceGrid
from paper_2309_04581_b200.scene import Camera, make_scene
from paper_2309_04581_b200.surface import Lambertian, Mirror, TriangleMesh
from paper_2309_04581_b200.transport import EstimationError, build_transport

pytestmark = pytest.mark.gpu


def _room(emission=(3.0, 2.0, 1.0), bsdf0=None):
    g = gs.load("transport.npz")
    meshes = [TriangleMesh(g["bv"], g["bf"], bsdf0 or Lambertian(np.full(3, 0.6))),
              TriangleMesh(g["qv"], g["qf"], Lambertian(np.array((0.2, 0.3, 0.4))),
                           emission=np.array(emission)),
              TriangleMesh(g["cv"], g["cf"], Lambertian(np.array((0.7, 0.5, 0.3))))]
    poses = [Camera(Transform.look_at([0, 0, 1.5], [0, 0, -1]), math.radians(60), (12, 10)),
             Camera(Transform.look_at([1.2, 0.8, 1.0], [0, -0.5, -1]), math.radians(50), (12, 10))]
    return make_scene(meshes=meshes, camera=poses[0], spp=4, seed=9, n_bounces=8), poses, g


def test_transport_matches_reference_golden():
    scene, poses, g = _room()
    op = build_transport(scene, poses, max_depth=3)
    assert op.a.shape == g["a"].shape == (2 * 12 * 10, 26, 3)
    assert np.array_equal(op.a != 0, g["a"] != 0)
    np.testing.assert_allclose(op.a, g["a"], rtol=1e-12, atol=1e-15)


def test_transport_is_linear_in_emission():
    scene, poses, _ = _room()
    op = build_transport(scene, poses, max_depth=3)
    e = np.zeros((op.n_faces, 3))
    e[12:14] = (3.0, 2.0, 1.0)                        # the emissive quad's two faces
    scene.render.n_bounces = 3
    img = renderer.render_surface_only(scene, camera=poses[1]).pixels
    np.testing.assert_allclose(op.images(e)[1].pixels, img, rtol=1e-12, atol=1e-14)


def test_transport_validation():
    scene, poses, _ = _room(bsdf0=Mirror(np.ones(3)))
    with pytest.raises(EstimationError):
        build_transport(scene, poses)
    scene, poses, _ = _room()
    with pytest.raises(EstimationError):
        build_transport(scene, [])
    scene.field = RadianceGrid.constant((-2,) * 3, (2,) * 3, 0.1, (0.1, 0.1, 0.1))
    with pytest.raises(EstimationError):
        build_transport(scene, poses)
