"""Ray/box and ray/triangle queries restated from the reference.

TEST INFRASTRUCTURE ONLY.

* `ray_slab`        - reference `field.py:88-101` (zero-direction handling).
* `moller_trumbore` - reference `surface.py:243-275`, same float64 operation
                      order, DET_EPS = 1e-12, BARY_EPS = 1e-7.
* `TriangleSet.nearest` / `.any_hit` - the hit contract of `Bvh.intersect_batch`
  / `any_hit_batch` / `brute_force_batch` (`surface.py:377-503`): strictly
  nearest t in (t_min, t_max], ties to the smaller face id. The acceleration
  structure here is the oracle's own (Morton-ordered buckets under an
  implicit binary tree, traversed breadth-first over (ray, node) pairs);
  the reference documents - and its tests check - that hits do not depend on
  the structure (`surface.py:5-7`, tests/test_surface.py:101-113).
"""

from __future__ import annotations

import numpy as np

BARY_EPS = 1e-7
DET_EPS = 1e-12


def ray_slab(lo, hi, o, d):
    """Entry/exit t of rays vs a box; empty overlap gives t0 > t1."""
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        ta = (lo - o) * inv
        tb = (hi - o) * inv
    flat = d == 0.0
    outside = (o < lo) | (o > hi)
    near = np.where(flat, np.where(outside, np.inf, -np.inf), np.minimum(ta, tb))
    far = np.where(flat, np.where(outside, -np.inf, np.inf), np.maximum(ta, tb))
    return near.max(axis=-1), far.min(axis=-1)


def moller_trumbore(o, d, v0, e1, e2, t_min, t_max):
    """t per broadcast (ray, face) pair, +inf where rejected."""
    dx, dy, dz = d[..., 0], d[..., 1], d[..., 2]
    ax, ay, az = e1[..., 0], e1[..., 1], e1[..., 2]
    bx, by, bz = e2[..., 0], e2[..., 1], e2[..., 2]
    px = dy * bz - dz * by
    py = dz * bx - dx * bz
    pz = dx * by - dy * bx
    det = ax * px + ay * py + az * pz
    good = np.abs(det) > DET_EPS
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / np.where(good, det, 1.0)
    sx = o[..., 0] - v0[..., 0]
    sy = o[..., 1] - v0[..., 1]
    sz = o[..., 2] - v0[..., 2]
    u = (sx * px + sy * py + sz * pz) * inv
    qx = sy * az - sz * ay
    qy = sz * ax - sx * az
    qz = sx * ay - sy * ax
    v = (dx * qx + dy * qy + dz * qz) * inv
    t = (bx * qx + by * qy + bz * qz) * inv
    ok = good & (u >= -BARY_EPS) & (v >= -BARY_EPS) & (u + v <= 1.0 + BARY_EPS) \
        & (t > t_min) & (t <= t_max)
    return np.where(ok, t, np.inf)


def _morton3(q):
    """30-bit Morton codes of (N,3) ints in [0, 1024)."""
    q = q.astype(np.uint64)
    out = np.zeros(len(q), np.uint64)
    for bit in range(10):
        for axis in range(3):
            out |= ((q[:, axis] >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit + axis)
    return out


class TriangleSet:
    """Faces (v0, e1, e2) in global-id order with an oracle-only tree."""

    BUCKET = 4

    def __init__(self, v0, e1, e2):
        self.v0, self.e1, self.e2 = (np.asarray(a, np.float64).reshape(-1, 3) for a in (v0, e1, e2))
        n = len(self.v0)
        self.n = n
        if n == 0:
            return
        v1 = self.v0 + self.e1
        v2 = self.v0 + self.e2
        lo = np.minimum(np.minimum(self.v0, v1), v2)
        hi = np.maximum(np.maximum(self.v0, v1), v2)
        # Moller-Trumbore accepts hits up to BARY_EPS outside a face, so the
        # boxes are padded to keep traversal equal to brute force.
        pad = 1e-6 * (hi - lo).max(axis=1, keepdims=True) + 1e-9 * (1.0 + np.abs(lo).max(axis=1, keepdims=True))
        lo, hi = lo - pad, hi + pad
        centre = 0.5 * (lo + hi)
        span = centre.max(0) - centre.min(0)
        q = np.floor((centre - centre.min(0)) / np.where(span > 0, span, 1.0) * 1023.0).astype(np.int64)
        self.order = np.argsort(_morton3(np.clip(q, 0, 1023)), kind="stable")
        n_leaf = -(-n // self.BUCKET)
        depth = max(0, int(np.ceil(np.log2(n_leaf))))
        self.depth = depth
        n_slots = 1 << depth
        blo = np.full((n_slots, 3), np.inf)
        bhi = np.full((n_slots, 3), -np.inf)
        slot = np.arange(n) // self.BUCKET
        np.minimum.at(blo, slot, lo[self.order])
        np.maximum.at(bhi, slot, hi[self.order])
        levels_lo, levels_hi = [blo], [bhi]
        for _ in range(depth):
            blo = np.minimum(blo[0::2], blo[1::2])
            bhi = np.maximum(bhi[0::2], bhi[1::2])
            levels_lo.append(blo)
            levels_hi.append(bhi)
        self.levels_lo = levels_lo[::-1]   # level 0 = root
        self.levels_hi = levels_hi[::-1]

    def _candidates(self, o, d, t_min, t_max):
        """(ray, face) pairs whose leaf box overlaps the ray interval."""
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = 1.0 / d
        rays = np.arange(len(o))
        nodes = np.zeros(len(o), np.int64)
        for lvl in range(self.depth + 1):
            lo, hi = self.levels_lo[lvl][nodes], self.levels_hi[lvl][nodes]
            with np.errstate(invalid="ignore"):
                ta = (lo - o[rays]) * inv[rays]
                tb = (hi - o[rays]) * inv[rays]
            near = np.where(np.isnan(ta) | np.isnan(tb), -np.inf, np.minimum(ta, tb)).max(1)
            far = np.where(np.isnan(ta) | np.isnan(tb), np.inf, np.maximum(ta, tb)).min(1)
            keep = (np.maximum(near, t_min[rays]) <= np.minimum(far, t_max[rays])) \
                & (lo <= hi).all(axis=1)
            rays, nodes = rays[keep], nodes[keep]
            if lvl < self.depth:
                rays = np.repeat(rays, 2)
                nodes = (np.repeat(nodes, 2) * 2 + np.tile([0, 1], len(nodes)))
        faces_r, faces_f = [], []
        for j in range(self.BUCKET):
            f = nodes * self.BUCKET + j
            ok = f < self.n
            faces_r.append(rays[ok])
            faces_f.append(self.order[f[ok]])
        return np.concatenate(faces_r), np.concatenate(faces_f)

    def _pair_t(self, o, d, r, f, t_min, t_max):
        return moller_trumbore(o[r], d[r], self.v0[f], self.e1[f], self.e2[f], t_min[r], t_max[r])

    def nearest(self, o, d, t_min=0.0, t_max=np.inf, chunk=1 << 15):
        """(t, face) per ray, face -1 / t inf on miss."""
        o = np.asarray(o, np.float64).reshape(-1, 3)
        d = np.asarray(d, np.float64).reshape(-1, 3)
        n = len(o)
        best_t = np.full(n, np.inf)
        best_f = np.full(n, -1, np.int64)
        if self.n == 0 or n == 0:
            return best_t, best_f
        tmin = np.broadcast_to(np.asarray(t_min, np.float64), (n,)).copy()
        tmax = np.broadcast_to(np.asarray(t_max, np.float64), (n,)).copy()
        for s in range(0, n, chunk):
            sl = slice(s, min(n, s + chunk))
            r, f = self._candidates(o[sl], d[sl], tmin[sl], tmax[sl])
            t = self._pair_t(o[sl], d[sl], r, f, tmin[sl], tmax[sl])
            hit = np.isfinite(t)
            r, f, t = r[hit], f[hit], t[hit]
            if not len(r):
                continue
            order = np.lexsort((f, t, r))
            r, f, t = r[order], f[order], t[order]
            first = np.ones(len(r), bool)
            first[1:] = r[1:] != r[:-1]
            best_t[s + r[first]] = t[first]
            best_f[s + r[first]] = f[first]
        return best_t, best_f

    def any_hit(self, o, d, t_min, t_max, chunk=1 << 15):
        o = np.asarray(o, np.float64).reshape(-1, 3)
        d = np.asarray(d, np.float64).reshape(-1, 3)
        n = len(o)
        blocked = np.zeros(n, bool)
        if self.n == 0 or n == 0:
            return blocked
        tmin = np.broadcast_to(np.asarray(t_min, np.float64), (n,)).copy()
        tmax = np.broadcast_to(np.asarray(t_max, np.float64), (n,)).copy()
        for s in range(0, n, chunk):
            sl = slice(s, min(n, s + chunk))
            r, f = self._candidates(o[sl], d[sl], tmin[sl], tmax[sl])
            t = self._pair_t(o[sl], d[sl], r, f, tmin[sl], tmax[sl])
            blocked[s + r[np.isfinite(t)]] = True
        return blocked

    def brute_nearest(self, o, d, t_min=0.0, t_max=np.inf):
        """All faces against all rays (the reference's oracle, surface.py:480-503)."""
        o = np.asarray(o, np.float64).reshape(-1, 3)
        d = np.asarray(d, np.float64).reshape(-1, 3)
        t = moller_trumbore(o[:, None], d[:, None], self.v0[None], self.e1[None], self.e2[None],
                            np.asarray(t_min)[..., None] if np.ndim(t_min) else t_min,
                            np.asarray(t_max)[..., None] if np.ndim(t_max) else t_max)
        k = np.argmin(t, axis=1)
        tk = t[np.arange(len(o)), k]
        return tk, np.where(np.isfinite(tk), k, -1)
