"""Field evaluation for the oracle.

TEST INFRASTRUCTURE ONLY.

`dense_sample` restates the reference field plugin `RadianceGrid.sample_batch`
(`field.py:143-161`) with `_trilinear` (`field.py:41-81`) and `_inside_mask`
(`field.py:84-85`) in the same float64 operation order.

`neural_*` is the CPU DEFINITION of the paper's hash-grid NeRF, which the
reference does not implement (parity against the reference is
unpinned, parity against this definition is what the GPU tests check):

* encode (bit-exact contract): p32 = float32(p_field); per level l and
  axis, x = (p32 - float32(lo)) * s_l (float32, two roundings), s_l =
  float32(N_l / (hi - lo)); i = clamp(floor(x), 0, N_l - 1); f = x - i.
  Corner c = (cx, cy, cz) = (c & 1, c >> 1 & 1, c >> 2) has weight
  (wx * wy) * wz with w = f or 1 - f, index dense  X + r*Y + r*r*Z (r = N_l+1)
  or hashed (X ^ Y*2654435761 ^ Z*805459861) & (T - 1) in uint32, and the
  feature is acc_0 + acc_1 where acc_x accumulates fma(w, table[...], acc_x)
  over the corners with cx = x in increasing c, in float32 from +0 (correctly
  rounded fused multiply-add; oracle/native.c pins it with glibc fmaf, the
  GPU uses fma.rn.f32x2 with the two x halves on the two lanes of a pair).
* MLP: float16 operands (features, hidden activations, weights), products
  exact, sums here in float64 (GPU: float32 tensor-core accumulation), ReLU
  then round-to-nearest float16 between layers; sigma = exp(z[0]);
  colour input = [SH16(d), z[1:16], 0]; sigmoid or softplus head.
* SH16: real spherical harmonics of bands 0-3 of the unit propagation
  direction in the field frame (standard published constants).
* occupancy: cell = clamp(floor((p32 - lo32) * float32(G / (hi - lo))), 0, G-1),
  bit x + G*(y + G*z) of uint32 words; a march sample is evaluated iff it is
  inside the box and its cell bit is set.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HASH_PY, HASH_PZ = np.uint64(2654435761), np.uint64(805459861)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def native():
    """ctypes handle on oracle/_build/liboracle.so (built on first use)."""
    global _LIB
    if _LIB is None:
        out = os.path.join(_HERE, "_build", "liboracle.so")
        src = os.path.join(_HERE, "native.c")
        if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
            os.makedirs(os.path.dirname(out), exist_ok=True)
            subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off",
                                   "-shared", "-fPIC", "-o", out, src, "-lm"])
        _LIB = ctypes.CDLL(out)
        _LIB.oracle_rotate_fma.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p]
        _LIB.oracle_corner_fma.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]
    return _LIB


def rotate_fma(v, rot):
    """Row-vectors v (N,3) through a 3x3 with the BLAS FMA chain."""
    v = np.ascontiguousarray(v, np.float64).reshape(-1, 3)
    rot = np.ascontiguousarray(rot, np.float64)
    out = np.empty_like(v)
    native().oracle_rotate_fma(len(v), v.ctypes.data, rot.ctypes.data, out.ctypes.data)
    return out


def corner_fma(w, v):
    """float32 (n, F): fma-accumulate 8 corner values v (n, 8, F) with
    weights w (n, 8) in corner order (exact, via glibc fmaf)."""
    w = np.ascontiguousarray(w, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    n, F = v.shape[0], v.shape[2]
    out = np.empty((n, F), np.float32)
    native().oracle_corner_fma(n, F, w.ctypes.data, v.ctypes.data, out.ctypes.data)
    return out


def to_field_frame(fp, p, d=None):
    """World -> field frame (reference field.py:148,171-174)."""
    if fp["identity"]:
        return p, d
    inv = fp["field_from_world"]
    pf = rotate_fma(p, inv[:3, :3]) + inv[:3, 3]
    return pf, (None if d is None else rotate_fma(d, inv[:3, :3]))


def inside_box(fp, pf):
    return ((pf >= fp["bbox_lo"]) & (pf <= fp["bbox_hi"])).all(axis=-1)


# --------------------------------------------------------------- dense grid

def _trilinear(values, lo, res, scale, p):
    g = (p - lo) * scale
    top = np.maximum(np.asarray(res, np.float64) - 1.0, 0.0)
    gc = np.clip(g, 0.0, np.maximum(top - 1e-9, 0.0))
    i0 = np.floor(gc).astype(np.int64)
    f = gc - i0
    i1 = np.minimum(i0 + 1, np.asarray(res) - 1)
    nx, ny, nz = res
    sx, sy = ny * nz, nz
    base = i0[:, 0] * sx + i0[:, 1] * sy + i0[:, 2]
    ox = (i1[:, 0] - i0[:, 0]) * sx
    oy = (i1[:, 1] - i0[:, 1]) * sy
    oz = i1[:, 2] - i0[:, 2]
    fx, fy, fz = f[:, 0:1], f[:, 1:2], f[:, 2:3]
    v = values.reshape(nx * ny * nz, -1)
    x00 = v[base] * (1 - fx) + v[base + ox] * fx
    x10 = v[base + oy] * (1 - fx) + v[base + ox + oy] * fx
    x01 = v[base + oz] * (1 - fx) + v[base + ox + oz] * fx
    x11 = v[base + oy + oz] * (1 - fx) + v[base + ox + oy + oz] * fx
    y0 = x00 * (1 - fy) + x10 * fy
    y1 = x01 * (1 - fy) + x11 * fy
    return y0 * (1 - fz) + y1 * fz


def dense_sample(fp, p):
    """(sigma (N,), rgb (N,3)) at world points, vacuum outside the box."""
    pf, _ = to_field_frame(fp, p)
    ins = inside_box(fp, pf)
    sigma = np.zeros(len(p))
    rgb = np.zeros((len(p), 3))
    if ins.any():
        q = pf[ins]
        res = tuple(int(r) for r in fp["res"])
        if fp["sigma_const"]:
            sigma[ins] = fp["sigma"][0]
        else:
            sigma[ins] = _trilinear(fp["sigma"], fp["bbox_lo"], res, fp["scale"], q)[:, 0]
        if fp["rad_const"]:
            rgb[ins] = fp["radiance"][0]
        else:
            rgb[ins] = _trilinear(fp["radiance"], fp["bbox_lo"], res, fp["scale"], q)
    return sigma, rgb


# ------------------------------------------------------------ neural field

def neural_encode(fp, pf, want_index=False):
    """float32 features (N, L*F) [and uint32 indices (N, L, 8)]."""
    n = len(pf)
    L, F = fp["n_levels"], fp["n_features"]
    mask = np.uint64((1 << fp["log2_table"]) - 1)
    p32 = pf.astype(np.float32)
    lo32 = fp["bbox_lo"].astype(np.float32)
    rel = p32 - lo32
    table = fp["table"]
    feat = np.zeros((n, L * F), np.float32)
    index = np.zeros((n, L, 8), np.uint32) if want_index else None
    one = np.float32(1.0)
    for lvl in range(L):
        nl = int(fp["level_n"][lvl])
        x = rel * fp["level_scale"][lvl]
        cell = np.clip(np.floor(x).astype(np.int64), 0, nl - 1)
        frac = x - cell.astype(np.float32)
        w_hi, w_lo = frac, one - frac
        r = nl + 1
        wts = np.empty((n, 8), np.float32)
        vals = np.empty((n, 8, F), np.float32)
        for c in range(8):
            bits = (c & 1, (c >> 1) & 1, c >> 2)
            w = [w_hi[:, a] if bits[a] else w_lo[:, a] for a in range(3)]
            wts[:, c] = (w[0] * w[1]) * w[2]
            cx, cy, cz = (cell[:, a] + bits[a] for a in range(3))
            if fp["level_dense"][lvl]:
                idx = (cx + r * cy + r * r * cz).astype(np.uint64)
            else:
                with np.errstate(over="ignore"):
                    idx = (cx.astype(np.uint64) ^ (cy.astype(np.uint64) * HASH_PY)
                           ^ (cz.astype(np.uint64) * HASH_PZ)) & mask
            vals[:, c] = table[int(fp["level_offset"][lvl]) + idx.astype(np.int64)]
            if want_index:
                index[:, lvl, c] = idx.astype(np.uint32)
        acc = corner_fma(wts, vals)
        feat[:, lvl * F:(lvl + 1) * F] = acc
    return (feat, index) if want_index else feat


SH_C = (0.28209479177387814, 0.4886025119029199, 1.0925484305920792,
        0.31539156525252005, 0.5462742152960396, 0.5900435899266435,
        2.890611442640554, 0.4570457994644658, 0.3731763325901154,
        1.445305721320277)


def sh16(d):
    """Real SH, bands 0..3, of unit directions (N,3) -> (N,16)."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    xx, yy, zz = x * x, y * y, z * z
    c = SH_C
    out = np.empty((len(d), 16))
    out[:, 0] = c[0]
    out[:, 1] = -c[1] * y
    out[:, 2] = c[1] * z
    out[:, 3] = -c[1] * x
    out[:, 4] = c[2] * x * y
    out[:, 5] = -c[2] * y * z
    out[:, 6] = c[3] * (3.0 * zz - 1.0)
    out[:, 7] = -c[2] * x * z
    out[:, 8] = c[4] * (xx - yy)
    out[:, 9] = -c[5] * y * (3.0 * xx - yy)
    out[:, 10] = c[6] * x * y * z
    out[:, 11] = -c[7] * y * (5.0 * zz - 1.0)
    out[:, 12] = c[8] * z * (5.0 * zz - 3.0)
    out[:, 13] = -c[7] * x * (5.0 * zz - 1.0)
    out[:, 14] = c[9] * z * (xx - yy)
    out[:, 15] = -c[5] * x * (xx - 3.0 * yy)
    return out


def _h(a):
    return np.asarray(a, np.float64).astype(np.float16).astype(np.float64)


def _layer(x16, w):
    return x16 @ w.astype(np.float64)


def neural_mlp(fp, feat, dfield, density_only=False):
    """(sigma f64 (N,), rgb f64 (N,3)) from features and field-frame dirs."""
    a1 = _h(np.maximum(_layer(_h(feat), fp["w_density1"]), 0.0))
    z2 = _layer(a1, fp["w_density2"])
    sigma = np.exp(z2[:, 0])
    if density_only:
        return sigma, None
    d32 = np.asarray(dfield, np.float64).astype(np.float32).astype(np.float64)
    cin = np.concatenate([sh16(d32), z2[:, 1:16], np.zeros((len(feat), 1))], axis=1)
    c1 = _h(np.maximum(_layer(_h(cin), fp["w_color1"]), 0.0))
    c2 = _h(np.maximum(_layer(c1, fp["w_color2"]), 0.0))
    c3 = _layer(c2, fp["w_color3"])
    if fp["act"] == 0:
        rgb = 1.0 / (1.0 + np.exp(-c3))
    else:
        rgb = np.where(c3 > 20.0, c3, np.log1p(np.exp(np.minimum(c3, 20.0))))
    return sigma, rgb


def occupancy_cell(fp, pf):
    g = int(fp["occ_res"])
    x = (pf.astype(np.float32) - fp["bbox_lo"].astype(np.float32)) * fp["occ_scale"]
    c = np.clip(np.floor(x).astype(np.int64), 0, g - 1)
    return c[:, 0] + g * (c[:, 1] + g * c[:, 2])


def occupancy_test(bits, cell):
    return ((bits[cell >> 5] >> (cell & 31).astype(np.uint32)) & np.uint32(1)).astype(bool)


def build_occupancy(fp, field_obj=None):
    """uint32 bitfield: cell occupied iff sigma(cell centre) > threshold."""
    g = int(fp["occ_res"])
    ijk = np.stack(np.meshgrid(np.arange(g), np.arange(g), np.arange(g), indexing="ij"), -1)
    ijk = ijk.transpose(2, 1, 0, 3).reshape(-1, 3).astype(np.float64)
    lo, hi = fp["bbox_lo"], fp["bbox_hi"]
    pf = lo + (ijk + 0.5) * ((hi - lo) / g)
    sigma, _ = neural_mlp(fp, neural_encode(fp, pf), None, density_only=True)
    occ = sigma > fp["occ_threshold"]
    words = np.zeros((g ** 3 + 31) // 32, np.uint32)
    idx = np.nonzero(occ)[0]
    np.bitwise_or.at(words, idx >> 5, (np.uint32(1) << (idx & 31).astype(np.uint32)))
    return words


def occupancy_bits(fp):
    if fp.get("occ_bits") is not None:
        return np.asarray(fp["occ_bits"], np.uint32)
    if "_occ_cache" not in fp:
        fp["_occ_cache"] = build_occupancy(fp)
    return fp["_occ_cache"]


def neural_sample(fp, p, d):
    """(sigma, rgb, evaluated) at world points; not evaluated = vacuum or
    empty occupancy cell (both contribute exactly nothing to the march)."""
    pf, df = to_field_frame(fp, p, d)
    n = len(p)
    ev = inside_box(fp, pf)
    if ev.any():
        ev[ev] = occupancy_test(occupancy_bits(fp), occupancy_cell(fp, pf[ev]))
    sigma = np.zeros(n)
    rgb = np.zeros((n, 3))
    if ev.any():
        s, c = neural_mlp(fp, neural_encode(fp, pf[ev]), df[ev])
        sigma[ev], rgb[ev] = s, c
    return sigma, rgb, ev
