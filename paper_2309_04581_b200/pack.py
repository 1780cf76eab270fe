"""Flatten a scene into the plain arrays the C-ABI (`include/hrt.h`) and the
CPU oracle both consume.

Accepts this package's `Scene` or a reference `hybridrt.scene.Scene`
(duck-typed on the attributes the reference renderer reads:
`render.py:204-246`, `scene.py:459-479`). Geometry is float64 and
world-space exactly as the reference stores it (`surface.py:160-161`,
`surface.py:301-313`): per-face v0, e1 = v1 - v0, e2 = v2 - v0, unit
normal, emission and mesh index, meshes concatenated in scene order (the
global face id). Shadow blockers are the non-emissive meshes, numbered
separately (`scene.py:540`).
"""

from __future__ import annotations

import math

import numpy as np

from .surface import material_record

FIELD_NONE, FIELD_DENSE, FIELD_NEURAL = 0, 1, 2


def _faces(meshes):
    tris, normals, emis, mesh_of = [], [], [], []
    for mi, m in enumerate(meshes):
        tv = np.asarray(m.vertices, np.float64)[np.asarray(m.indices)]
        tris.append(tv)
        normals.append(np.asarray(m.face_normals, np.float64))
        e = m.emission if m.emission is not None else np.zeros((len(tv), 3))
        emis.append(np.asarray(e, np.float64))
        mesh_of.append(np.full(len(tv), mi, np.int32))
    if not tris:
        z = np.zeros((0, 3))
        return z.reshape(0, 3, 3), z, z.copy(), np.zeros(0, np.int32)
    return (np.concatenate(tris), np.concatenate(normals),
            np.concatenate(emis), np.concatenate(mesh_of))


def _edges(tri):
    return (np.ascontiguousarray(tri[:, 0]), np.ascontiguousarray(tri[:, 1] - tri[:, 0]),
            np.ascontiguousarray(tri[:, 2] - tri[:, 0]))


def _is_emissive(m):
    return m.emission is not None and bool(np.any(np.asarray(m.emission) > 0))


def _transform_arrays(wff):
    m = np.asarray(wff.m, np.float64)
    ident = bool(m[0, 0] == 1.0 and m[1, 1] == 1.0 and m[2, 2] == 1.0 and not m[:3, 3].any()
                 and not m[0, 1:3].any() and not m[1, 0::2].any() and not m[2, 0:2].any())
    return ident, np.ascontiguousarray(wff.m_inv, np.float64)


def pack_field(field) -> dict:
    if field is None:
        return {"kind": FIELD_NONE}
    ident, inv = _transform_arrays(field.world_from_field)
    out = {"bbox_lo": np.asarray(field.bbox_lo, np.float64),
           "bbox_hi": np.asarray(field.bbox_hi, np.float64),
           "identity": ident, "field_from_world": inv}
    if getattr(field, "kind", None) == "neural":
        out.update(
            kind=FIELD_NEURAL, n_levels=field.n_levels, n_features=field.n_features,
            log2_table=field.log2_table, enc_dim=field.enc_dim,
            level_n=field.level_n.astype(np.int32), level_offset=field.level_offset.astype(np.int64),
            level_dense=field.level_dense.astype(np.int32), level_scale=field.level_scales(),
            table=field.table, w_density1=field.w_density1, w_density2=field.w_density2,
            w_color1=field.w_color1, w_color2=field.w_color2, w_color3=field.w_color3,
            act=field.act_code, occ_res=field.occupancy_res,
            occ_threshold=field.occupancy_threshold, occ_scale=field.occupancy_scale(),
            occ_bits=field.occupancy_bits)
        return out
    # Dense RadianceGrid: C-order (z fastest) node arrays, as `_trilinear`
    # flattens them (reference field.py:41-81).
    sigma = np.ascontiguousarray(field.sigma, np.float64)
    rad = np.ascontiguousarray(field.radiance, np.float64)
    res = tuple(int(v) for v in sigma.shape)
    scale = np.array([(r - 1) / (h - l) if r > 1 else 0.0
                      for r, l, h in zip(res, out["bbox_lo"], out["bbox_hi"])])
    s_flat = sigma.reshape(-1)
    r_flat = rad.reshape(-1, 3)
    out.update(kind=FIELD_DENSE, res=np.array(res, np.int32), scale=scale,
               sigma=s_flat, radiance=r_flat,
               sigma_const=bool((s_flat == s_flat[0]).all()),
               rad_const=bool((r_flat == r_flat[0]).all()))
    return out


def pack_scene(scene) -> dict:
    meshes = list(scene.meshes)
    tri, normal, emission, mesh_of = _faces(meshes)
    v0, e1, e2 = _edges(tri)
    blockers = [m for m in meshes if not _is_emissive(m)]
    btri = _faces(blockers)[0]
    bv0, be1, be2 = _edges(btri)
    mats = [material_record(m.bsdf) for m in meshes]
    rc = scene.render
    em = scene.emitters
    if em is not None and len(em) > 0:
        emit = {"tris": np.ascontiguousarray(em.triangles, np.float64).reshape(-1, 9),
                "cdf": np.asarray(em.cdf, np.float64), "r_src": np.asarray(em.r_src, np.float64)}
    else:
        emit = {"tris": np.zeros((0, 9)), "cdf": np.zeros(0), "r_src": np.zeros(0)}
    return {
        "v0": v0, "e1": e1, "e2": e2, "normal": np.ascontiguousarray(normal),
        "emission": np.ascontiguousarray(emission), "mesh_of": mesh_of,
        "mat_kind": np.array([k for k, _, _ in mats], np.int32),
        "mat_rgb": np.array([c for _, c, _ in mats], np.float64).reshape(-1, 3),
        "mat_ior": np.array([i for _, _, i in mats], np.float64),
        "bv0": bv0, "be1": be1, "be2": be2,
        "emitters": emit,
        "field": pack_field(scene.field),
        "n_bounces": int(rc.n_bounces), "threshold": float(rc.threshold),
        "march_step": float(rc.march_step), "spawn_eps": float(scene.spawn_eps),
        "sample_cap": int(getattr(rc, "sample_cap", 0) or 0),
        "early_t": float(getattr(rc, "early_t", 0.0) or 0.0),
    }


def pack_camera(camera) -> dict:
    """Pose rotation/position and the scalars `Camera.primary_rays` uses
    (reference render.py:61-74): tan(fov/2) via numpy, aspect = w/h."""
    w, h = camera.resolution
    m = np.asarray(camera.pose.m, np.float64)
    return {"rot": np.ascontiguousarray(m[:3, :3]), "pos": np.ascontiguousarray(m[:3, 3]),
            "tan_half": float(np.tan(0.5 * camera.fov)), "aspect": w / h,
            "width": int(w), "height": int(h)}


def stratify_k(spp: int) -> int:
    """k for k x k stratified jitter when spp = k^2 > 1 else 0 (render.py:320-330)."""
    k = int(math.floor(math.sqrt(spp)))
    return k if (k * k == spp and k > 1) else 0
