"""The render path restated on the CPU (numpy, float64).

TEST INFRASTRUCTURE ONLY. Consumes the packed scene/camera dicts from
`paper_2309_04581_b200.pack` (plain arrays, so this module never calls the
product). Functions follow the reference line by line in semantics:

* `primary_rays`   - render.py:61-74 (+ core.py:183-187 via the FMA chain)
* `sample_jitter`  - render.py:320-330
* `march`          - render.py:142-172 + field.py:218-255, plus the NeRF
                     additions of SURVEY P4/P5 (occupancy filter, per-path
                     sample cap, in-march early-out; all off for dense grids
                     unless the RenderConfig enables them)
* `shadow_mask`    - render.py:96-123 (EmitterSet.sample + any-hit)
* `bsdf_sample`    - render.py:175-201 + surface.py:74-121
* `trace_paths`    - render.py:204-246 (and the degenerate tracers 249-299)
* `render`         - render.py:333-380 (per-pixel sum in sample order, / spp)
"""

from __future__ import annotations

import numpy as np

from . import rng
from .field import dense_sample, neural_sample, occupancy_cell, rotate_fma, to_field_frame
from .geometry import TriangleSet, ray_slab

SHADOW_SHRINK = 1.0 - 1e-4
MASK_FLOOR = 0.02
FIELD_NONE, FIELD_DENSE, FIELD_NEURAL = 0, 1, 2
MAT_LAMBERTIAN, MAT_MIRROR, MAT_DIELECTRIC = 0, 1, 2


def _dot(a, b):
    return (a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1]) + a[:, 2] * b[:, 2]


def _norm(a):
    return np.sqrt((a[:, 0] * a[:, 0] + a[:, 1] * a[:, 1]) + a[:, 2] * a[:, 2])


def _cross(a, b):
    return np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
                     a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                     a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)


class OracleScene:
    def __init__(self, pack):
        self.pack = pack
        self.tris = TriangleSet(pack["v0"], pack["e1"], pack["e2"])
        self.blockers = TriangleSet(pack["bv0"], pack["be1"], pack["be2"])
        self.field = pack["field"]
        self.em = pack["emitters"]


# ------------------------------------------------------------- camera rays

def primary_rays(cam, pix, jx, jy):
    w, h = cam["width"], cam["height"]
    i = pix % w
    j = pix // w
    x = (2.0 * (i + jx) / w - 1.0) * cam["tan_half"] * cam["aspect"]
    y = (1.0 - 2.0 * (j + jy) / h) * cam["tan_half"]
    dw = rotate_fma(np.stack([x, y, -np.ones_like(x)], axis=1), cam["rot"])
    dw = dw / _norm(dw)[:, None]
    o = np.broadcast_to(cam["pos"], dw.shape).copy()
    return o, dw


def stratify_k(spp):
    k = int(np.floor(np.sqrt(spp)))
    return k if (k * k == spp and k > 1) else 0


def sample_jitter(seed, pix, smp, spp):
    u1 = rng.uniform(seed, pix, smp, 0, rng.PIXEL_X, 0)
    u2 = rng.uniform(seed, pix, smp, 0, rng.PIXEL_Y, 0)
    k = stratify_k(spp)
    if k:
        return (smp % k + u1) / k, (smp // k + u2) / k
    return u1, u2


# ------------------------------------------------------------------ shadows

def shadow_mask(sc, p, seed, pix, smp, bounce, lane):
    em = sc.em
    if len(em["cdf"]) == 0:
        return np.ones(len(p))
    u_pick = rng.uniform(seed, pix, smp, bounce, rng.LIGHT_PICK, lane)
    u1 = rng.uniform(seed, pix, smp, bounce, rng.LIGHT_U, lane)
    u2 = rng.uniform(seed, pix, smp, bounce, rng.LIGHT_V, lane)
    n_em = len(em["cdf"])
    idx = np.minimum(np.searchsorted(em["cdf"], u_pick, side="right"), n_em - 1)
    tri = em["tris"][idx].reshape(-1, 3, 3)
    su = np.sqrt(u1)
    b0, b1, b2 = 1.0 - su, su * (1.0 - u2), su * u2
    q = b0[:, None] * tri[:, 0] + b1[:, None] * tri[:, 1] + b2[:, None] * tri[:, 2]
    delta = q - p
    dist = _norm(delta)
    d = delta / np.maximum(dist, 1e-12)[:, None]
    blocked = sc.blockers.any_hit(p, d, sc.pack["spawn_eps"], dist * SHADOW_SHRINK)
    masked = np.clip(1.0 - em["r_src"][idx], MASK_FLOOR, 1.0)
    return np.where(blocked, masked, 1.0)


# ------------------------------------------------------------------- march

def field_bounds(fp, o, d):
    if fp["identity"]:
        return ray_slab(fp["bbox_lo"], fp["bbox_hi"], o, d)
    of, df = to_field_frame(fp, o, d)
    return ray_slab(fp["bbox_lo"], fp["bbox_hi"], of, df)


def march(sc, ids, o, d, s_end, bounce, pix, smp, seed, st, trace=None):
    """Advance st['L'], st['Ts'], st['T'], st['neval'] of paths `ids` over
    their field segment [max(t0, 0), min(t1, s_end)]."""
    fp = sc.field
    pk = sc.pack
    t0, t1 = field_bounds(fp, o[ids], d[ids])
    s0 = np.maximum(t0, 0.0)
    s1 = np.minimum(t1, s_end)
    go = s1 > s0
    if not go.any():
        return
    ids, s0, s1 = ids[go], s0[go], s1[go]
    seg = np.maximum(s1 - s0, 0.0)
    dt = pk["march_step"]
    n = np.ceil(seg / dt).astype(np.int64)
    n = np.where(seg > 0.0, np.maximum(n, 1), 0)
    cap, early = pk["sample_cap"], pk["early_t"]
    halted = np.zeros(len(ids), bool)
    neural = fp["kind"] == FIELD_NEURAL
    shadows = len(sc.em["cdf"]) > 0
    L, Ts, T, nev = st["L"], st["Ts"], st["T"], st["neval"]
    for k in range(int(n.max())):
        act = (k < n) & ~halted
        if not act.any():
            break
        if early > 0:
            low = act & (Ts[ids].max(axis=1) < early)
            halted |= low
            act &= ~low
        loc = np.nonzero(act)[0]
        sel = ids[loc]
        delta = seg[loc] / n[loc]
        t_mid = s0[loc] + (k + 0.5) * delta
        p = o[sel] + t_mid[:, None] * d[sel]
        if neural:
            sigma, rad, ev = neural_sample(fp, p, d[sel])
        else:
            sigma, rad = dense_sample(fp, p)
            ev = np.ones(len(sel), bool)
        if cap > 0:
            over = ev & (nev[sel] >= cap)
            halted[loc[over]] = True
            ev &= ~over
            sigma = np.where(ev, sigma, 0.0)
            rad = np.where(ev[:, None], rad, 0.0)
        nev[sel] += ev
        if trace is not None and neural and ev.any():
            pf, _ = to_field_frame(fp, p[ev])
            trace.append((sel[ev], np.full(ev.sum(), bounce), np.full(ev.sum(), k),
                          occupancy_cell(fp, pf)))
        a = 1.0 - np.exp(-sigma * delta)
        m = 1.0
        if shadows:
            need = (a > 0.0) & (rad.max(axis=1) > 0.0)
            if need.any():
                st["nshadow"] = st.get("nshadow", 0) + int(need.sum())
                m = np.ones(len(a))
                m[need] = shadow_mask(sc, p[need], seed, pix[sel[need]], smp[sel[need]],
                                      bounce, k)
        L[sel] += Ts[sel] * (a * m)[:, None] * rad
        keep = 1.0 - a
        Ts[sel] *= keep[:, None]
        T[sel] *= keep


# ------------------------------------------------------------------- BSDFs

def _reflect(wo, n):
    return 2.0 * _dot(wo, n)[:, None] * n - wo


def _cosine(n, u1, u2):
    a = np.where(np.abs(n[:, 0:1]) > 0.9, [0.0, 1.0, 0.0], [1.0, 0.0, 0.0])
    t = _cross(a, n)
    t = t / _norm(t)[:, None]
    b = _cross(n, t)
    phi = 2.0 * np.pi * u1
    sin_t = np.sqrt(u2)
    z = np.sqrt(1.0 - u2)
    lx = np.cos(phi) * sin_t
    ly = np.sin(phi) * sin_t
    return lx[:, None] * t + ly[:, None] * b + z[:, None] * n


def _dielectric(wo, n, front, ior, u):
    cos_i = np.clip(_dot(wo, n), 0.0, 1.0)
    eta = np.where(front, 1.0 / ior, ior)
    sin2_t = eta * eta * np.maximum(1.0 - cos_i * cos_i, 0.0)
    tir = sin2_t > 1.0
    r0 = ((ior - 1.0) / (ior + 1.0)) ** 2
    p_refl = r0 + (1.0 - r0) * np.power(1.0 - cos_i, 5)
    reflect = tir | (u < p_refl)
    refl = _reflect(wo, n)
    cos_t = np.sqrt(np.maximum(1.0 - sin2_t, 0.0))
    refr = eta[:, None] * (-wo) + (eta * cos_i - cos_t)[:, None] * n
    rn = _norm(refr)[:, None]
    refr = refr / np.where(rn > 0, rn, 1.0)
    return np.where(reflect[:, None], refl, refr)


def bsdf_sample(sc, faces, wo, n, front, pix, smp, bounce, seed):
    pk = sc.pack
    mat = pk["mesh_of"][faces]
    kind = pk["mat_kind"][mat]
    new_d = np.zeros((len(faces), 3))
    weight = pk["mat_rgb"][mat].copy()
    for code in np.unique(kind):
        s = kind == code
        if code == MAT_LAMBERTIAN:
            u1 = rng.uniform(seed, pix[s], smp[s], bounce, rng.BSDF_U, 0)
            u2 = rng.uniform(seed, pix[s], smp[s], bounce, rng.BSDF_V, 0)
            new_d[s] = _cosine(n[s], u1, u2)
        elif code == MAT_MIRROR:
            new_d[s] = _reflect(wo[s], n[s])
        else:
            for mi in np.unique(mat[s]):
                s2 = s & (mat == mi)
                u = rng.uniform(seed, pix[s2], smp[s2], bounce, rng.BSDF_LOBE, 0)
                new_d[s2] = _dielectric(wo[s2], n[s2], front[s2], float(pk["mat_ior"][mi]), u)
    return new_d, weight


# -------------------------------------------------------------- bounce loop

def new_state(n):
    return {"L": np.zeros((n, 3)), "Ts": np.ones((n, 3)), "T": np.ones(n),
            "neval": np.zeros(n, np.int64)}


def trace_paths(sc, o, d, pix, smp, seed, mode="hybrid", st=None, trace=None, hits=None):
    """Linear radiance (N,3) of camera paths; mode 'hybrid' | 'surface' | 'volume'."""
    pk = sc.pack
    n = len(o)
    st = st or new_state(n)
    has_field = sc.field["kind"] != FIELD_NONE
    if mode == "volume":
        if has_field:
            march(sc, np.arange(n), o, d, np.full(n, np.inf), 1, pix, smp, seed, st, trace)
        return st["L"]
    ro, rd = o.copy(), d.copy()
    alive = np.arange(n)
    for bounce in range(1, pk["n_bounces"] + 1):
        if not len(alive):
            break
        t_hit, face = sc.tris.nearest(ro[alive], rd[alive])
        if hits is not None:
            hits.append((alive.copy(), np.full(len(alive), bounce), t_hit, face))
        if has_field and mode == "hybrid":
            march(sc, alive, ro, rd, t_hit, bounce, pix, smp, seed, st, trace)
        hit = face >= 0
        hid = alive[hit]
        if not len(hid):
            break
        f = face[hit]
        point = ro[hid] + t_hit[hit][:, None] * rd[hid]
        n_raw = pk["normal"][f]
        facing = _dot(n_raw, rd[hid]) < 0.0
        normal = np.where(facing[:, None], n_raw, -n_raw)
        st["L"][hid] += st["Ts"][hid] * np.where(facing[:, None], pk["emission"][f], 0.0)
        new_d, weight = bsdf_sample(sc, f, -rd[hid], normal, facing, pix[hid], smp[hid],
                                    bounce, seed)
        st["Ts"][hid] *= weight
        ro[hid] = point + pk["spawn_eps"] * new_d
        rd[hid] = new_d
        alive = hid[st["Ts"][hid].max(axis=1) >= pk["threshold"]]
    assert not np.isnan(st["L"]).any(), "NaN radiance in path batch"
    return st["L"]


def render(pack, cam, spp, seed, pixels=None, mode="hybrid", stats=None, trace=None):
    """(h, w, 3) float64 image, or (len(pixels), 3) for a pixel subset.
    Path p of pixel q has sample index p % spp; per-pixel sums run in sample
    order, then divide by spp (render.py:339-350)."""
    if spp < 1:
        raise ValueError("spp must be >= 1")
    sc = pack if isinstance(pack, OracleScene) else OracleScene(pack)
    w, h = cam["width"], cam["height"]
    pix_list = np.arange(w * h) if pixels is None else np.asarray(pixels, np.int64)
    pix = np.repeat(pix_list, spp)
    smp = np.tile(np.arange(spp), len(pix_list))
    jx, jy = sample_jitter(seed, pix, smp, spp)
    o, d = primary_rays(cam, pix, jx, jy)
    st = new_state(len(pix))
    L = trace_paths(sc, o, d, pix, smp, seed, mode=mode, st=st, trace=trace)
    # per-pixel sums grouped as the reference's batches (render.py:333-350):
    # a 16-row band of npix = rows * w pixels takes max(1, 65536 // npix)
    # samples per batch, each batch summed with .sum(axis=1), then added
    acc = np.zeros((len(pix_list), 3))
    Lr = L.reshape(len(pix_list), spp, 3)
    row = pix_list // w
    band = row - row % 16
    per_batch = np.maximum(1, 65536 // (np.minimum(16, h - band) * w))
    for pb in np.unique(per_batch):
        sel = per_batch == pb
        s = 0
        while s < spp:
            sb = min(int(pb), spp - s)
            acc[sel] += Lr[sel, s:s + sb].sum(axis=1)
            s += sb
    out = acc / spp
    if stats is not None:
        stats["nerf_samples"] = int(st["neval"].sum())
        stats["paths"] = len(pix)
        stats["shadow_rays"] = int(st.get("nshadow", 0))
    assert np.isfinite(out).all() and (out >= 0.0).all()
    return out.reshape(h, w, 3) if pixels is None else out
