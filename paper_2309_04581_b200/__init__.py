"""B200-native hybrid NeRF/mesh renderer (arXiv 2309.04581), drop-in for the
reference `hybridrt` render path.

Public names mirror the reference package's render/scene subset
(reference `hybridrt/__init__.py:6-37`). Rendering always runs in the
sm_100a kernels of libhrt.so; importing the render functions without a
built library or a CUDA device raises instead of falling back to the CPU.
"""

__version__ = "0.1.0"

from .core import Ray, Transform, tone_map
from .field import NeuralField, RadianceGrid
from .images import HdrImage, decode_pfm, decode_ppm, encode_pfm, encode_ppm
from .scene import Camera, EmitterSet, RenderConfig, Scene, make_scene, scene_diagonal
from .surface import Dielectric, Lambertian, Mirror, TriangleMesh
from .rng import PathRng
from .nerffile import load_nerf, load_scene, save_nerf

_RENDER_NAMES = ("render", "render_surface_only", "render_volume_only", "trace_path", "finalize",
                 "Renderer", "renderer_for")


def __getattr__(name):
    # torch + libhrt.so are loaded on first use of the render path only, so
    # host-side scene construction works in a CPU-only process.
    if name in _RENDER_NAMES:
        from . import renderer as _render
        return getattr(_render, name)
    raise AttributeError(name)


__all__ = ["Ray", "Transform", "tone_map", "NeuralField", "RadianceGrid", "HdrImage",
           "decode_pfm", "decode_ppm", "encode_pfm", "encode_ppm", "Camera", "EmitterSet",
           "RenderConfig", "Scene", "make_scene", "scene_diagonal", "Dielectric", "Lambertian",
           "Mirror", "TriangleMesh", "PathRng", "load_nerf", "load_scene", "save_nerf", *_RENDER_NAMES]
