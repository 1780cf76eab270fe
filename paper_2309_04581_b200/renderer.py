"""Drop-in render entry points (reference `hybridrt/render.py:302-401`).

`render(scene, camera=None, spp=None, seed=None, threads=1) -> HdrImage`
keeps the reference signature, argument meaning and errors (ValueError for
spp < 1, AssertionError for non-finite/negative radiance) and accepts either
this package's `Scene` or a reference `hybridrt.scene.Scene`. The scene is
packed and uploaded once per (scene, geometry version) into a native
`hrt_handle`; every frame then runs entirely in the sm_100a kernels of
libhrt.so (include/hrt.h). `threads` is accepted for API compatibility;
GPU work has no host thread pool.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .images import HdrImage
from .pack import pack_camera, pack_scene, stratify_k  # noqa: F401  (re-export)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Renderer:
    """One uploaded scene on the current CUDA device."""

    def __init__(self, scene_or_pack):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2309_04581_b200 renders on CUDA (sm_100a) only; no CPU path")
        self.lib = _lib.load()
        self.pack = scene_or_pack if isinstance(scene_or_pack, dict) else pack_scene(scene_or_pack)
        keep = _lib._Keep()
        desc = _lib.scene_desc(self.pack, keep)
        handle = ctypes.c_void_p()
        _lib.check(self.lib.hrt_create(ctypes.byref(desc), ctypes.byref(handle)), "hrt_create")
        self.handle = handle
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.last_stats = {}
        self.config = _config_of(self.pack)

    def set_config(self, config):
        """(n_bounces, threshold, march_step, spawn_eps, sample_cap, early_t) for later renders."""
        if tuple(config) != self.config:
            _lib.check(self.lib.hrt_set_config(self.handle, *config), "hrt_set_config")
            self.config = tuple(config)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.hrt_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ frames
    def render_pixels(self, camera, spp, seed, mode=_lib.MODE_HYBRID, pixels=None, out=None,
                      frame_ptr=None):
        """(n, 3) float64 device tensor for `pixels` (int32 device tensor of
        pixel ids, None = whole frame in raster order). With `frame_ptr` (a
        device address of a raster (w*h, 3) float64 frame, e.g. a peer GPU's
        mapped with tiles.PeerFrame) the pixels are stored there by pixel id
        instead (HRT_OUT_BY_PIXEL) and None is returned."""
        if spp < 1:
            raise ValueError("spp must be >= 1")
        cam = _lib.camera_desc(camera if isinstance(camera, dict) else pack_camera(camera))
        n = cam.width * cam.height if pixels is None else int(pixels.numel())
        if frame_ptr is not None:
            out_ptr, mode = ctypes.c_void_p(int(frame_ptr)), int(mode) | _lib.OUT_BY_PIXEL
        else:
            if out is None:
                out = torch.empty((n, 3), dtype=torch.float64, device=self.device)
            out_ptr = _dptr(out)
        if n == 0:                                   # a rank without tiles
            self.last_stats = _lib.Stats().as_dict()
            return out
        stats = _lib.Stats()
        rc = self.lib.hrt_render(self.handle, ctypes.byref(cam), int(spp), int(seed) & (2**64 - 1),
                                 int(mode), _dptr(pixels), n, out_ptr, ctypes.byref(stats),
                                 _stream())
        self.last_stats = stats.as_dict()
        _lib.check(rc, "hrt_render")
        return out

    @staticmethod
    def pinned(shape, dtype):
        """A numpy array in page-locked host memory (render_host DMAs it
        directly; the array keeps its pinned storage alive)."""
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()

    def render_host(self, camera, spp, seed, mode=_lib.MODE_HYBRID, pixels=None, out=None):
        """Same through host buffers (numpy in/out, copies inside the call;
        page-locked buffers, see `pinned`, are DMA'd without staging)."""
        cam = _lib.camera_desc(camera if isinstance(camera, dict) else pack_camera(camera))
        pix = None if pixels is None else np.ascontiguousarray(pixels, np.int32)
        n = cam.width * cam.height if pix is None else len(pix)
        if out is None:
            out = np.empty((n, 3), np.float64)
        stats = _lib.Stats()
        rc = self.lib.hrt_render_host(self.handle, ctypes.byref(cam), int(spp),
                                      int(seed) & (2**64 - 1), int(mode),
                                      None if pix is None else pix.ctypes.data_as(ctypes.c_void_p),
                                      n, out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(stats))
        self.last_stats = stats.as_dict()
        _lib.check(rc, "hrt_render_host")
        return out

    def trace(self, o, d, pixel, sample, seed, mode=_lib.MODE_HYBRID):
        """L (n,3) of caller rays (device tensors)."""
        n = o.shape[0]
        L = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        rc = self.lib.hrt_trace_paths(self.handle, _dptr(o), _dptr(d), _dptr(pixel), _dptr(sample),
                                      n, int(seed) & (2**64 - 1), int(mode), _dptr(L), _stream())
        _lib.check(rc, "hrt_trace_paths")
        return L

    def refit(self, scene):
        pk = pack_scene(scene)
        if len(pk["v0"]) != len(self.pack["v0"]) or len(pk["bv0"]) != len(self.pack["bv0"]):
            raise ValueError("refit needs the same topology; build a new Renderer")
        arrs = [np.ascontiguousarray(pk[k], np.float64) for k in
                ("v0", "e1", "e2", "normal", "bv0", "be1", "be2")]
        ptrs = [a.ctypes.data_as(ctypes.c_void_p) if a.size else None for a in arrs]
        _lib.check(self.lib.hrt_refit(self.handle, *ptrs), "hrt_refit")
        self.pack = pk

    def set_field_transform(self, field):
        """Upload a moved field's placement (hrt_set_field_transform)."""
        from .pack import _transform_arrays
        ident, inv = _transform_arrays(field.world_from_field)
        inv = np.ascontiguousarray(inv, np.float64).reshape(16)
        _lib.check(self.lib.hrt_set_field_transform(self.handle, int(ident), inv.ctypes.data_as(ctypes.c_void_p)),
                   "hrt_set_field_transform")
        self.pack["field"]["identity"] = ident
        self.pack["field"]["field_from_world"] = inv.reshape(4, 4)

    def set_rigid_base(self, object_vertices, indices, emissive=None):
        """Object-space geometry for refit_rigid: per mesh (in scene order) its
        object vertices and faces; `emissive` flags exclude meshes from the
        blocker tree as pack_scene does."""
        corners = np.concatenate([np.asarray(v, np.float64)[np.asarray(f).reshape(-1, 3)].reshape(-1, 9)
                                  for v, f in zip(object_vertices, indices)])
        emissive = emissive or [False] * len(indices)
        blk, base = [], 0
        for f, e in zip(indices, emissive):
            nf = len(np.asarray(f).reshape(-1, 3))
            if not e:
                blk.append(np.arange(base, base + nf, dtype=np.int32))
            base += nf
        blk = np.concatenate(blk) if blk else np.zeros(0, np.int32)
        if len(corners) != len(self.pack["v0"]) or len(blk) != len(self.pack["bv0"]):
            raise ValueError("rigid base does not match the scene's faces")
        corners = np.ascontiguousarray(corners)
        self._rigid_keep = (corners, blk)
        _lib.check(self.lib.hrt_set_rigid_base(self.handle, corners.ctypes.data_as(ctypes.c_void_p),
                                               blk.ctypes.data_as(ctypes.c_void_p)), "hrt_set_rigid_base")

    def refit_rigid(self, transforms):
        """Move every mesh by its 3x4 world_from_object (n_meshes, 3, 4) and
        refit both trees on the GPU (hrt_refit_rigid)."""
        xf = np.ascontiguousarray(transforms, np.float64).reshape(-1, 12)
        _lib.check(self.lib.hrt_refit_rigid(self.handle, xf.ctypes.data_as(ctypes.c_void_p), len(xf)),
                   "hrt_refit_rigid")

    # ------------------------------------------------------------ probes
    def field_sample(self, points, dirs=None, use_occupancy=False):
        n = points.shape[0]
        sigma = torch.empty(n, dtype=torch.float32, device=self.device)
        rgb = torch.empty((n, 3), dtype=torch.float32, device=self.device) if dirs is not None else None
        ev = torch.empty(n, dtype=torch.int32, device=self.device)
        rc = self.lib.hrt_field_sample(self.handle, _dptr(points), _dptr(dirs), n, _dptr(sigma),
                                       _dptr(rgb), _dptr(ev), int(use_occupancy), _stream())
        _lib.check(rc, "hrt_field_sample")
        return sigma, rgb, ev

    def field_encode(self, points, with_index=True):
        fp = self.pack["field"]
        n = points.shape[0]
        feat = torch.empty((n, fp["enc_dim"]), dtype=torch.float32, device=self.device)
        idx = (torch.empty((n, fp["n_levels"], 8), dtype=torch.int32, device=self.device)
               if with_index else None)
        rc = self.lib.hrt_field_encode(self.handle, _dptr(points), n, _dptr(feat), _dptr(idx),
                                       _stream())
        _lib.check(rc, "hrt_field_encode")
        return feat, idx

    def occupancy(self):
        g = self.pack["field"]["occ_res"]
        words = np.zeros((g ** 3 + 31) // 32, np.uint32)
        _lib.check(self.lib.hrt_occupancy(self.handle, words.ctypes.data_as(ctypes.c_void_p),
                                          len(words)), "hrt_occupancy")
        return words

    def intersect(self, o, d, t_min=None, t_max=None, blocker=False, any_hit=False):
        n = o.shape[0]
        if any_hit:
            hit = torch.empty(n, dtype=torch.uint8, device=self.device)
            rc = self.lib.hrt_intersect(self.handle, int(blocker), 1, _dptr(o), _dptr(d),
                                        _dptr(t_min), _dptr(t_max), n, None, None, _dptr(hit),
                                        _stream())
            _lib.check(rc, "hrt_intersect")
            return hit.bool()
        t = torch.empty(n, dtype=torch.float64, device=self.device)
        f = torch.empty(n, dtype=torch.int64, device=self.device)
        rc = self.lib.hrt_intersect(self.handle, int(blocker), 0, _dptr(o), _dptr(d), _dptr(t_min),
                                    _dptr(t_max), n, _dptr(t), _dptr(f), None, _stream())
        _lib.check(rc, "hrt_intersect")
        return t, f

    def set_march(self, continuous=True):
        """Continuous wavefront march (default) or the reference's bounce-by-bounce loop."""
        _lib.check(self.lib.hrt_set_march(self.handle, int(bool(continuous))), "hrt_set_march")

    def set_profile(self, on=True):
        """Per-stage device timing of later renders (last_stats['stage_ms'])."""
        _lib.check(self.lib.hrt_set_profile(self.handle, int(bool(on))), "hrt_set_profile")

    def gather_peak(self, mode=2):
        """Measured random one-entry gather rate (useful GB/s; 8-B entries for
        F = 2, 16-B for F = 4) over this scene's hash table: the roofline of
        the encode (hrt_gather_peak)."""
        v = ctypes.c_double(0.0)
        _lib.check(self.lib.hrt_gather_peak(self.handle, int(mode), ctypes.byref(v)), "hrt_gather_peak")
        return v.value

    def round_rows(self, cap=1024):
        """(rows, samples, field_ms) per device-driven march round of the last
        render (hrt_round_rows): batch rows (holes included), the samples in
        them, and the field-engine time."""
        rows = np.zeros(cap, np.int64)
        smp = np.zeros(cap, np.int64)
        ms = np.zeros(cap, np.float32)
        n = ctypes.c_int32(0)
        _lib.check(self.lib.hrt_round_rows(self.handle, rows.ctypes.data_as(ctypes.c_void_p),
                                           smp.ctypes.data_as(ctypes.c_void_p),
                                           ms.ctypes.data_as(ctypes.c_void_p), cap, ctypes.byref(n)),
                   "hrt_round_rows")
        return rows[:n.value], smp[:n.value], ms[:n.value]

    def l2_peak(self):
        """Measured L2 roofline over this scene's hash table (hrt_l2_peak):
        coalesced read GB/s and random 32-B sector-gather GB/s."""
        rd, sec, nb = ctypes.c_double(0.0), ctypes.c_double(0.0), ctypes.c_int64(0)
        _lib.check(self.lib.hrt_l2_peak(self.handle, ctypes.byref(rd), ctypes.byref(sec), ctypes.byref(nb)),
                   "hrt_l2_peak")
        return {"read_gbs": rd.value, "gather_sector_gbs": sec.value, "bytes": nb.value}

    def set_trace(self, records, cap):
        _lib.check(self.lib.hrt_set_trace(self.handle, _dptr(records), int(cap)), "hrt_set_trace")


def uniform_keys(keys):
    """rng.uniform over an (n, 6) int64 device tensor of key tuples."""
    lib = _lib.load()
    out = torch.empty(keys.shape[0], dtype=torch.float64, device=keys.device)
    _lib.check(lib.hrt_uniform(_dptr(keys), keys.shape[0], _dptr(out), _stream()), "hrt_uniform")
    return out


def primary_rays(camera, pixel, sample, seed, spp):
    lib = _lib.load()
    cam = _lib.camera_desc(camera if isinstance(camera, dict) else pack_camera(camera))
    n = pixel.shape[0]
    o = torch.empty((n, 3), dtype=torch.float64, device=pixel.device)
    d = torch.empty((n, 3), dtype=torch.float64, device=pixel.device)
    _lib.check(lib.hrt_primary_rays(ctypes.byref(cam), _dptr(pixel), _dptr(sample), n,
                                    int(seed) & (2**64 - 1), int(spp), _dptr(o), _dptr(d),
                                    _stream()), "hrt_primary_rays")
    return o, d


# ------------------------------------------------------------------ cache

def _field_key(scene):
    """The field placement the handle must use (reference dynamic fields move
    by reassigning world_from_field between frames, sim.py:673-698, with no
    BVH rebuild)."""
    f = getattr(scene, "field", None)
    if f is None:
        return None
    return np.asarray(f.world_from_field.m, np.float64).tobytes()


def _config_of(pack):
    return (int(pack["n_bounces"]), float(pack["threshold"]), float(pack["march_step"]),
            float(pack["spawn_eps"]), int(pack["sample_cap"]), float(pack["early_t"]))


def _scene_config(scene, spawn_eps):
    rc = scene.render
    return (int(rc.n_bounces), float(rc.threshold), float(rc.march_step), float(spawn_eps),
            int(getattr(rc, "sample_cap", 0) or 0), float(getattr(rc, "early_t", 0.0) or 0.0))


class _Cached:
    """A scene's renderer plus what it was uploaded from: this package's
    `Scene.version`, the reference Scene's Bvh OBJECT (held, compared with
    `is`: `rebuild_bvh` swaps it, and an id() could be reused once the old
    one is freed) and the field placement bytes."""

    def __init__(self, scene, r, dev):
        self.r, self.dev = r, dev
        self.stamp(scene)

    def stamp(self, scene):
        self.version = getattr(scene, "version", None)
        self.bvh = getattr(scene, "bvh", None)
        self.field = _field_key(scene)

    def geometry_changed(self, scene):
        return getattr(scene, "version", None) != self.version or getattr(scene, "bvh", None) is not self.bvh


def renderer_for(scene) -> Renderer:
    """The scene's cached renderer: geometry changes refit, a moved field
    re-uploads its placement (hrt_set_field_transform), RenderConfig changes
    (read at every call, as the reference does) are pushed with
    hrt_set_config."""
    cached = getattr(scene, "_hrt_renderer", None)
    dev = torch.cuda.current_device()
    if cached is not None and cached.dev == dev:
        r = cached.r
        if cached.geometry_changed(scene):
            r.refit(scene)
        fk = _field_key(scene)
        if fk != cached.field:
            r.set_field_transform(scene.field)
        cached.stamp(scene)
    else:
        r = Renderer(scene)
        scene._hrt_renderer = _Cached(scene, r, dev)
    r.set_config(_scene_config(scene, r.pack["spawn_eps"]))
    return r


def _image(scene, pixels):
    """`hybridrt.images.HdrImage` for a reference Scene (so the reference's
    render and this one return the same type), else this package's."""
    if type(scene).__module__.startswith("hybridrt"):
        import sys
        mod = sys.modules.get("hybridrt.images")
        if mod is not None:
            return mod.HdrImage(pixels)
    return HdrImage(pixels)


def _resolve(scene, camera, spp, seed):
    camera = camera or scene.camera
    spp = scene.render.spp if spp is None else int(spp)
    seed = scene.render.seed if seed is None else int(seed)
    if spp < 1:
        raise ValueError("spp must be >= 1")
    return camera, spp, seed


def _frame(scene, camera, spp, seed, mode):
    camera, spp, seed = _resolve(scene, camera, spp, seed)
    r = renderer_for(scene)
    out = r.render_pixels(camera, spp, seed, mode)
    w, h = camera.resolution
    return _image(scene, out.cpu().numpy().reshape(h, w, 3))


def render(scene, camera=None, spp=None, seed=None, threads=1) -> HdrImage:
    """Average spp hybrid paths per pixel into a linear HDR image (render.py:372-380)."""
    return _frame(scene, camera, spp, seed, _lib.MODE_HYBRID)


def render_surface_only(scene, camera=None, spp=None, seed=None, threads=1) -> HdrImage:
    """Degeneracy reference A: no volume marching (render.py:383-388)."""
    return _frame(scene, camera, spp, seed, _lib.MODE_SURFACE)


def render_volume_only(scene, camera=None, spp=None, seed=None, threads=1) -> HdrImage:
    """Degeneracy reference B: one full-field march per camera ray (render.py:391-396)."""
    return _frame(scene, camera, spp, seed, _lib.MODE_VOLUME)


def trace_path(ray, scene, path_rng) -> np.ndarray:
    """Linear radiance of one camera path keyed (seed, pixel, sample) (render.py:302-312)."""
    r = renderer_for(scene)
    dev = r.device
    o = torch.tensor(np.asarray(ray.origin, np.float64).reshape(1, 3), device=dev)
    d = torch.tensor(np.asarray(ray.dir, np.float64).reshape(1, 3), device=dev)
    pix = torch.tensor([int(path_rng.pixel)], dtype=torch.int64, device=dev)
    smp = torch.tensor([int(path_rng.sample)], dtype=torch.int64, device=dev)
    return r.trace(o, d, pix, smp, int(path_rng.seed)).cpu().numpy()[0]


def finalize_device(src, width, height, hdr_output, pixel=None):
    """K9 on the device: encoded PFM / PPM bytes (uint8 CUDA tensor) of float64
    radiance rows `src` (n, 3); `pixel` (int32, < 0 = padding) gives each
    row's global pixel id, None means `src` is the raster frame
    (hrt_finalize)."""
    lib = _lib.load()
    src = src.contiguous()
    n = int(src.shape[0])
    nb = ctypes.c_int64(0)
    args = (int(width), int(height), _dptr(src), _dptr(pixel) if pixel is not None else None, n,
            int(bool(hdr_output)))
    _lib.check(lib.hrt_finalize(*args, None, 0, ctypes.byref(nb), _stream()), "hrt_finalize")
    out = torch.empty(nb.value, dtype=torch.uint8, device=src.device)
    _lib.check(lib.hrt_finalize(*args, _dptr(out), nb.value, ctypes.byref(nb), _stream()),
               "hrt_finalize")
    return out


def finalize(img: HdrImage, hdr_output: bool) -> bytes:
    """PFM bytes for HDR output, else tone-mapped 8-bit PPM (render.py:399-401),
    encoded on the GPU (K9)."""
    px = torch.as_tensor(np.ascontiguousarray(img.pixels, np.float64).reshape(-1, 3), device="cuda")
    return finalize_device(px, img.w, img.h, hdr_output).cpu().numpy().tobytes()
