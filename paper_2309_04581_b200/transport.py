"""Transport operator for emitter estimation on the GPU (reference
`hybridrt/emitters.py:47-166`): `build_transport(scene, poses, max_depth)`
renders every pose once with surface-only Lambertian paths that scatter their
throughput into per-face bins (hrt_transport), so image = A @ emission
exactly. Checks, errors and the returned `TransportOperator` mirror the
reference; the estimation loop itself (loss / gradient descent / pruning)
is out of scope."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .images import HdrImage
from .pack import material_record

TRANSPORT_BYTE_CAP = 1_500_000_000      # emitters.py:24


class EstimationError(ValueError):
    pass


@dataclass
class TransportOperator:
    """Dense per-channel transport: image_c = A[..., c] @ E[:, c] (emitters.py:47-70)."""

    a: np.ndarray            # (poses*h*w, faces, 3)
    n_poses: int
    resolution: tuple        # (w, h)
    n_faces: int
    spp: int
    seed: int

    def apply(self, emission: np.ndarray) -> np.ndarray:
        return np.einsum("rfc,fc->rc", self.a, emission)

    def images(self, emission: np.ndarray) -> list:
        w, h = self.resolution
        flat = self.apply(emission)
        return [HdrImage(flat[i * h * w:(i + 1) * h * w].reshape(h, w, 3))
                for i in range(self.n_poses)]


def build_transport(scene, poses, max_depth: int = 3) -> TransportOperator:
    """emitters.py:114-166 on the GPU: same validation, same operator."""
    import torch

    from . import _lib
    from .pack import pack_camera
    from .renderer import _dptr, _stream, renderer_for

    for m in scene.meshes:
        if material_record(m.bsdf)[0] != 0:
            raise EstimationError(
                f"estimation requires Lambertian surfaces; mesh '{getattr(m, 'name', '?')}' is not")
    if scene.field is not None:
        raise EstimationError("estimation scenes must not contain a radiance field")
    n_faces = int(sum(len(np.asarray(m.indices).reshape(-1, 3)) for m in scene.meshes))
    if not poses:
        raise EstimationError("at least one pose required")
    w, h = poses[0].resolution
    rows = len(poses) * h * w
    need = rows * n_faces * 3 * 8
    if need > TRANSPORT_BYTE_CAP:
        raise EstimationError(
            f"dense transport operator would need {need / 1e9:.1f} GB "
            f"({rows} rows x {n_faces} faces); reduce faces/resolution or "
            "use finite-difference gradients")
    for cam in poses:
        if tuple(cam.resolution) != (w, h):
            raise EstimationError("all poses must share one resolution")
    spp, seed = int(scene.render.spp), int(scene.render.seed)
    r = renderer_for(scene)
    cams = (_lib.CameraDesc * len(poses))(*[_lib.camera_desc(pack_camera(c)) for c in poses])
    out = torch.empty((rows, n_faces, 3), dtype=torch.float64, device=r.device)
    _lib.check(r.lib.hrt_transport(r.handle, ctypes.cast(cams, ctypes.c_void_p), len(poses), spp,
                                   ctypes.c_uint64(seed), int(max_depth), _dptr(out), _stream()),
               "hrt_transport")
    return TransportOperator(a=out.cpu().numpy(), n_poses=len(poses), resolution=(w, h),
                             n_faces=n_faces, spp=spp, seed=seed)
