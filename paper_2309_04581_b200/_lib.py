"""ctypes binding of the C ABI in include/hrt.h (libhrt.so, built in-tree).

There is deliberately no fallback: if the shared library is missing or was
built for another architecture, importing the render path raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HRT_LIB", os.path.join(_HERE, "libhrt.so"))

HRT_OK, HRT_EINVAL, HRT_ENONFINITE, HRT_ECUDA, HRT_ENOMEM = range(5)
MODE_HYBRID, MODE_SURFACE, MODE_VOLUME = 0, 1, 2
OUT_BY_PIXEL = 0x100

c_double_p = ctypes.POINTER(ctypes.c_double)
c_float_p = ctypes.POINTER(ctypes.c_float)
c_i32_p = ctypes.POINTER(ctypes.c_int32)
c_i64_p = ctypes.POINTER(ctypes.c_int64)
c_u16_p = ctypes.POINTER(ctypes.c_uint16)
c_u32_p = ctypes.POINTER(ctypes.c_uint32)
vp = ctypes.c_void_p


class FieldDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("identity", ctypes.c_int32),
        ("bbox_lo", ctypes.c_double * 3), ("bbox_hi", ctypes.c_double * 3),
        ("field_from_world", ctypes.c_double * 16),
        ("res", ctypes.c_int32 * 3), ("scale", ctypes.c_double * 3),
        ("sigma", c_double_p), ("radiance", c_double_p),
        ("sigma_const", ctypes.c_int32), ("rad_const", ctypes.c_int32),
        ("n_levels", ctypes.c_int32), ("n_features", ctypes.c_int32),
        ("log2_table", ctypes.c_int32), ("act", ctypes.c_int32),
        ("level_n", c_i32_p), ("level_offset", c_i64_p), ("level_dense", c_i32_p),
        ("level_scale", c_float_p), ("table", c_float_p), ("n_entries", ctypes.c_int64),
        ("w_density1", c_u16_p), ("w_density2", c_u16_p), ("w_color1", c_u16_p),
        ("w_color2", c_u16_p), ("w_color3", c_u16_p),
        ("occ_res", ctypes.c_int32), ("occ_scale", ctypes.c_float * 3),
        ("occ_threshold", ctypes.c_double), ("occ_bits", c_u32_p),
    ]


class SceneDesc(ctypes.Structure):
    _fields_ = [
        ("n_faces", ctypes.c_int64),
        ("v0", c_double_p), ("e1", c_double_p), ("e2", c_double_p),
        ("normal", c_double_p), ("emission", c_double_p), ("mesh_of", c_i32_p),
        ("n_materials", ctypes.c_int32), ("mat_kind", c_i32_p), ("mat_rgb", c_double_p),
        ("mat_ior", c_double_p),
        ("n_blockers", ctypes.c_int64), ("bv0", c_double_p), ("be1", c_double_p),
        ("be2", c_double_p),
        ("n_emitters", ctypes.c_int32), ("emitter_tris", c_double_p),
        ("emitter_cdf", c_double_p), ("emitter_rsrc", c_double_p),
        ("field", FieldDesc),
        ("n_bounces", ctypes.c_int32), ("threshold", ctypes.c_double),
        ("march_step", ctypes.c_double), ("spawn_eps", ctypes.c_double),
        ("sample_cap", ctypes.c_int32), ("early_t", ctypes.c_double),
    ]


class CameraDesc(ctypes.Structure):
    _fields_ = [("rot", ctypes.c_double * 9), ("pos", ctypes.c_double * 3),
                ("tan_half", ctypes.c_double), ("aspect", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("paths", ctypes.c_int64), ("nerf_samples", ctypes.c_int64),
                ("shadow_rays", ctypes.c_int64), ("bounce_rays", ctypes.c_int64),
                ("trace_records", ctypes.c_int64), ("ms", ctypes.c_float),
                ("field_ms", ctypes.c_float), ("field_launches", ctypes.c_int32),
                ("launches", ctypes.c_int64), ("evaluated", ctypes.c_int64),
                ("rounds", ctypes.c_int64), ("stage_ms", ctypes.c_float * 8),
                ("batch_rows", ctypes.c_int64), ("shadow_traced", ctypes.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["stage_ms"] = dict(zip(STAGES, list(self.stage_ms)))
        return d


# hrt.h HRT_STAGE_* order
STAGES = ("raygen", "intersect", "march_gen", "field", "shadow", "composite", "shade", "accumulate")


# name -> (restype, argtypes); this list is what include/hrt.h declares.
SIGNATURES = {
    "hrt_last_error": (ctypes.c_char_p, []),
    "hrt_version": (ctypes.c_int, []),
    "hrt_create": (ctypes.c_int, [ctypes.POINTER(SceneDesc), ctypes.POINTER(vp)]),
    "hrt_destroy": (ctypes.c_int, [vp]),
    "hrt_render": (ctypes.c_int, [vp, ctypes.POINTER(CameraDesc), ctypes.c_int32, ctypes.c_uint64,
                                  ctypes.c_int32, vp, ctypes.c_int64, vp, ctypes.POINTER(Stats), vp]),
    "hrt_render_host": (ctypes.c_int, [vp, ctypes.POINTER(CameraDesc), ctypes.c_int32,
                                       ctypes.c_uint64, ctypes.c_int32, vp, ctypes.c_int64, vp,
                                       ctypes.POINTER(Stats)]),
    "hrt_trace_paths": (ctypes.c_int, [vp, vp, vp, vp, vp, ctypes.c_int64, ctypes.c_uint64,
                                       ctypes.c_int32, vp, vp]),
    "hrt_set_trace": (ctypes.c_int, [vp, vp, ctypes.c_int64]),
    "hrt_set_profile": (ctypes.c_int, [vp, ctypes.c_int32]),
    "hrt_set_march": (ctypes.c_int, [vp, ctypes.c_int32]),
    "hrt_set_config": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int32, ctypes.c_double]),
    "hrt_finalize": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, vp, vp, ctypes.c_int64, ctypes.c_int32,
                                    vp, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), vp]),
    "hrt_transport": (ctypes.c_int, [vp, vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                     ctypes.c_int32, vp, vp]),
    "hrt_set_rigid_base": (ctypes.c_int, [vp, vp, vp]),
    "hrt_refit_rigid": (ctypes.c_int, [vp, vp, ctypes.c_int32]),
    "hrt_buffer_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(vp)]),
    "hrt_buffer_free": (ctypes.c_int, [vp]),
    "hrt_ipc_handle": (ctypes.c_int, [vp, vp]),
    "hrt_ipc_open": (ctypes.c_int, [vp, ctypes.POINTER(vp)]),
    "hrt_ipc_close": (ctypes.c_int, [vp]),
    "hrt_gather_peak": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]),
    "hrt_set_field_transform": (ctypes.c_int, [vp, ctypes.c_int32, vp]),
    "hrt_round_rows": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]),
    "hrt_l2_peak": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int64)]),
    "hrt_refit": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "hrt_field_sample": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int32, vp]),
    "hrt_field_encode": (ctypes.c_int, [vp, vp, ctypes.c_int64, vp, vp, vp]),
    "hrt_occupancy": (ctypes.c_int, [vp, vp, ctypes.c_int64]),
    "hrt_intersect": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp,
                                     ctypes.c_int64, vp, vp, vp, vp]),
    "hrt_uniform": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp]),
    "hrt_primary_rays": (ctypes.c_int, [ctypes.POINTER(CameraDesc), vp, vp, ctypes.c_int64,
                                        ctypes.c_uint64, ctypes.c_int32, vp, vp, vp]),
}

_lib = None


def load():
    """The loaded library (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (nvcc, sm_100a)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str = "hrt"):
    if rc == HRT_OK:
        return
    msg = f"{what}: {load().hrt_last_error().decode(errors='replace')}"
    if rc == HRT_EINVAL:
        raise ValueError(msg)
    if rc == HRT_ENONFINITE:
        raise AssertionError(msg)
    raise RuntimeError(msg)


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))


class _Keep(list):
    """Keeps host arrays alive while a descriptor points at them."""

    def arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.append(a)
        return a


def field_desc(fp: dict, keep: _Keep) -> FieldDesc:
    fd = FieldDesc()
    fd.kind = fp["kind"]
    if fp["kind"] == 0:
        fd.identity = 1
        return fd
    fd.identity = int(fp["identity"])
    fd.bbox_lo[:] = list(fp["bbox_lo"])
    fd.bbox_hi[:] = list(fp["bbox_hi"])
    fd.field_from_world[:] = list(np.asarray(fp["field_from_world"], np.float64).reshape(16))
    if fp["kind"] == 1:
        fd.res[:] = [int(v) for v in fp["res"]]
        fd.scale[:] = [float(v) for v in fp["scale"]]
        fd.sigma = _ptr(keep.arr(fp["sigma"], np.float64), ctypes.c_double)
        fd.radiance = _ptr(keep.arr(fp["radiance"], np.float64), ctypes.c_double)
        fd.sigma_const = int(fp["sigma_const"])
        fd.rad_const = int(fp["rad_const"])
        return fd
    fd.n_levels, fd.n_features = fp["n_levels"], fp["n_features"]
    fd.log2_table, fd.act = fp["log2_table"], fp["act"]
    fd.level_n = _ptr(keep.arr(fp["level_n"], np.int32), ctypes.c_int32)
    fd.level_offset = _ptr(keep.arr(fp["level_offset"], np.int64), ctypes.c_int64)
    fd.level_dense = _ptr(keep.arr(fp["level_dense"], np.int32), ctypes.c_int32)
    fd.level_scale = _ptr(keep.arr(fp["level_scale"], np.float32), ctypes.c_float)
    table = keep.arr(fp["table"], np.float32)
    fd.table = _ptr(table, ctypes.c_float)
    fd.n_entries = table.shape[0]
    for name in ("w_density1", "w_density2", "w_color1", "w_color2", "w_color3"):
        bits = keep.arr(np.asarray(fp[name], np.float16).view(np.uint16), np.uint16)
        setattr(fd, name, _ptr(bits, ctypes.c_uint16))
    fd.occ_res = fp["occ_res"]
    fd.occ_scale[:] = [float(v) for v in np.asarray(fp["occ_scale"], np.float32)]
    fd.occ_threshold = fp["occ_threshold"]
    if fp.get("occ_bits") is not None:
        fd.occ_bits = _ptr(keep.arr(fp["occ_bits"], np.uint32), ctypes.c_uint32)
    return fd


def scene_desc(pk: dict, keep: _Keep) -> SceneDesc:
    d = SceneDesc()
    d.n_faces = len(pk["v0"])
    for name in ("v0", "e1", "e2", "normal", "emission"):
        setattr(d, name, _ptr(keep.arr(pk[name], np.float64), ctypes.c_double))
    d.mesh_of = _ptr(keep.arr(pk["mesh_of"], np.int32), ctypes.c_int32)
    d.n_materials = len(pk["mat_kind"])
    d.mat_kind = _ptr(keep.arr(pk["mat_kind"], np.int32), ctypes.c_int32)
    d.mat_rgb = _ptr(keep.arr(pk["mat_rgb"], np.float64), ctypes.c_double)
    d.mat_ior = _ptr(keep.arr(pk["mat_ior"], np.float64), ctypes.c_double)
    d.n_blockers = len(pk["bv0"])
    for name in ("bv0", "be1", "be2"):
        setattr(d, name, _ptr(keep.arr(pk[name], np.float64), ctypes.c_double))
    em = pk["emitters"]
    d.n_emitters = len(em["cdf"])
    d.emitter_tris = _ptr(keep.arr(em["tris"], np.float64), ctypes.c_double)
    d.emitter_cdf = _ptr(keep.arr(em["cdf"], np.float64), ctypes.c_double)
    d.emitter_rsrc = _ptr(keep.arr(em["r_src"], np.float64), ctypes.c_double)
    d.field = field_desc(pk["field"], keep)
    d.n_bounces, d.threshold = pk["n_bounces"], pk["threshold"]
    d.march_step, d.spawn_eps = pk["march_step"], pk["spawn_eps"]
    d.sample_cap, d.early_t = pk["sample_cap"], pk["early_t"]
    return d


def camera_desc(cp: dict) -> CameraDesc:
    c = CameraDesc()
    c.rot[:] = list(np.asarray(cp["rot"], np.float64).reshape(9))
    c.pos[:] = list(np.asarray(cp["pos"], np.float64))
    c.tan_half, c.aspect = cp["tan_half"], cp["aspect"]
    c.width, c.height = cp["width"], cp["height"]
    return c
