"""Transport-operator timing: GPU build_transport on a
Lambertian room (3 meshes, 26 faces) at 64x64, 4 poses, 16 spp, depth 3.
With --reference (this container only: needs /root/reference) the reference
CPU build_transport on the same scene is timed instead."""
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")

RES, POSES, SPP = (64, 64), 4, 16


def scene_parts(mod_assets):
    bv, bf = mod_assets.box((-2, -2, -2), (2, 2, 2), inward=True)
    qv, qf = mod_assets.quad((-1, -1, -1.9), (2, 0, 0), (0, 2, 0))
    cv, cf = mod_assets.box((-0.5, -1.5, -1.0), (0.3, -0.4, 0.2))
    return (bv, bf), (qv, qf), (cv, cf)


def poses_of(Camera, Transform):
    return [Camera(Transform.look_at([1.2 * math.cos(k), 0.5, 1.2 * math.sin(k) + 0.3], [0, -0.5, -1]),
                   math.radians(55), RES) for k in range(POSES)]


if "--reference" in sys.argv:
    sys.path.insert(0, "/root/reference/pkg/src")
    from hybridrt import assets
    from hybridrt.core import Transform
    from hybridrt.emitters import build_transport
    from hybridrt.render import Camera
    from hybridrt.surface import Lambertian, TriangleMesh
    from golden.make_golden import make_scene
else:
    import torch
    from paper_2309_04581_b200 import assets
    from paper_2309_04581_b200.core import Transform
    from paper_2309_04581_b200.scene import Camera, make_scene
    from paper_2309_04581_b200.surface import Lambertian, TriangleMesh
    from paper_2309_04581_b200.transport import build_transport

(bv, bf), (qv, qf), (cv, cf) = scene_parts(assets)
meshes = [TriangleMesh(bv, bf, Lambertian(np.full(3, 0.6))),
          TriangleMesh(qv, qf, Lambertian(np.array((0.2, 0.3, 0.4))), emission=np.array((3.0, 2.0, 1.0))),
          TriangleMesh(cv, cf, Lambertian(np.array((0.7, 0.5, 0.3))))]
poses = poses_of(Camera, Transform)
scene = make_scene(meshes=meshes, camera=poses[0], spp=SPP, seed=9, n_bounces=8)
build_transport(scene, poses[:1], max_depth=3)           # warm
t = time.perf_counter()
op = build_transport(scene, poses, max_depth=3)
dt = time.perf_counter() - t
paths = POSES * RES[0] * RES[1] * SPP
print(f"{'reference CPU' if '--reference' in sys.argv else 'GPU'} build_transport: {dt*1e3:.1f} ms for "
      f"{paths} paths ({paths/dt/1e6:.3f} M paths/s), A {op.a.shape}, sum {op.a.sum():.6f}")
