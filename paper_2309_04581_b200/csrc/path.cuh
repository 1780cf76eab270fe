// path.cuh - per-path device functions of the bounce loop: camera rays (K1),
// dense-grid field lookups, shadow masks (K3), BSDF sampling and spawn (K8).
// Every function follows the cited reference lines in float64 operation
// order (build uses --fmad=false; reference-side fusions use __fma_rn).
#pragma once
#include "bvh.cuh"
#include "common.cuh"

namespace path {

struct Camera {
    double rot[9];
    double pos[3];
    double tan_half, aspect;
    int32_t width, height;
};

// render.py:320-330 (_sample_jitter) + render.py:61-74 (primary_rays).
HRT_DEV void primary_ray(const Camera& c, int64_t pix, int64_t smp, uint64_t seed, int32_t strat,
                         d3& o, d3& d) {
    double jx = rng::uniform(seed, pix, smp, 0, rng::PIXEL_X, 0);
    double jy = rng::uniform(seed, pix, smp, 0, rng::PIXEL_Y, 0);
    if (strat > 1) {
        jx = ((double)(smp % strat) + jx) / (double)strat;
        jy = ((double)(smp / strat) + jy) / (double)strat;
    }
    const int64_t i = pix % c.width, j = pix / c.width;
    const double x = ((2.0 * ((double)i + jx) / (double)c.width - 1.0) * c.tan_half) * c.aspect;
    const double y = (1.0 - 2.0 * ((double)j + jy) / (double)c.height) * c.tan_half;
    const double z = -1.0;
    // OpenBLAS order of (N,3) @ R^T: fma(x2, r2, fma(x1, r1, x0 * r0))
    d3 w = {__fma_rn(z, c.rot[2], __fma_rn(y, c.rot[1], x * c.rot[0])),
            __fma_rn(z, c.rot[5], __fma_rn(y, c.rot[4], x * c.rot[3])),
            __fma_rn(z, c.rot[8], __fma_rn(y, c.rot[7], x * c.rot[6]))};
    const double n = norm(w);
    d = {w.x / n, w.y / n, w.z / n};
    o = {c.pos[0], c.pos[1], c.pos[2]};
}

// -------------------------------------------------------------- dense grid
// field.py:41-81 (_trilinear) for one point and one channel group.
struct Trilerp {
    int64_t base, ox, oy, oz;
    double fx, fy, fz;
};

HRT_DEV Trilerp trilerp_setup(const DevField& f, d3 pf) {
    const DenseGrid& g = f.dense;
    const double p[3] = {pf.x, pf.y, pf.z};
    int64_t i0[3], i1[3];
    double fr[3];
    for (int a = 0; a < 3; ++a) {
        const double gg = (p[a] - f.lo[a]) * g.scale[a];
        const double top = fmax((double)g.res[a] - 1.0, 0.0);
        const double gc = fmin(fmax(gg, 0.0), fmax(top - 1e-9, 0.0));
        const double fl = floor(gc);
        i0[a] = (int64_t)fl;
        fr[a] = gc - (double)i0[a];
        i1[a] = min(i0[a] + 1, (int64_t)g.res[a] - 1);
    }
    const int64_t sx = (int64_t)g.res[1] * g.res[2], sy = g.res[2];
    return {i0[0] * sx + i0[1] * sy + i0[2], (i1[0] - i0[0]) * sx, (i1[1] - i0[1]) * sy,
            i1[2] - i0[2], fr[0], fr[1], fr[2]};
}

HRT_DEV double trilerp(const double* v, int C, int c, const Trilerp& t) {
    auto at = [&](int64_t i) { return __ldg(v + i * C + c); };
    const double gx = 1 - t.fx, gy = 1 - t.fy, gz = 1 - t.fz;
    const double x00 = at(t.base) * gx + at(t.base + t.ox) * t.fx;
    const double x10 = at(t.base + t.oy) * gx + at(t.base + t.ox + t.oy) * t.fx;
    const double x01 = at(t.base + t.oz) * gx + at(t.base + t.ox + t.oz) * t.fx;
    const double x11 = at(t.base + t.oy + t.oz) * gx + at(t.base + t.ox + t.oy + t.oz) * t.fx;
    const double y0 = x00 * gy + x10 * t.fy;
    const double y1 = x01 * gy + x11 * t.fy;
    return y0 * gz + y1 * t.fz;
}

// RadianceGrid.sample_batch (field.py:143-161) for one world point.
HRT_DEV double dense_sample(const DevField& f, d3 p, double rgb[3]) {
    const d3 pf = field_point(f, p);
    rgb[0] = rgb[1] = rgb[2] = 0.0;
    if (!inside_box(f.lo, f.hi, pf)) return 0.0;
    const DenseGrid& g = f.dense;
    Trilerp t;
    if (!g.sigma_const || !g.rad_const) t = trilerp_setup(f, pf);
    double s;
    if (g.sigma_const) s = g.sigma0;
    else s = trilerp(g.sigma, 1, 0, t);
    for (int c = 0; c < 3; ++c) rgb[c] = g.rad_const ? g.rad0[c] : trilerp(g.rad, 3, c, t);
    return s;
}

// ----------------------------------------------------------------- shadows
// EmitterSet.sample + shadow_mask_batch (render.py:96-123) for one point:
// 0 if the sampled emitter point is visible, else 1 + emitter index.
struct ShadowRay {          // one shadow query: point p towards emitter idx, interval (eps, tmax]
    d3 dir;
    double tmax;
    int32_t idx;
    double su, u2;          // the light sample's (sqrt(u1), u2) (shadow entry table patch)
};

// EmitterSet.sample (render.py:96-107) + the ray set-up of shadow_mask_batch
// (render.py:110-123) for one point.
// h4 = rng::prefix(seed, pix, smp, bounce) of the path segment.
HRT_DEV ShadowRay shadow_ray_h(const DevScene& sc, d3 p, uint64_t h4, int64_t lane) {
    const DevEmitters& em = sc.em;
    const double u_pick = rng::uniform_from(h4, rng::LIGHT_PICK, lane);
    const double u1 = rng::uniform_from(h4, rng::LIGHT_U, lane);
    const double u2 = rng::uniform_from(h4, rng::LIGHT_V, lane);
    int lo = 0, hi = em.n;            // searchsorted(cdf, u, 'right')
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (em.cdf[mid] <= u_pick) lo = mid + 1; else hi = mid;
    }
    const int idx = min(lo, em.n - 1);
    const double* t = em.tris + 9 * idx;
    const double su = sqrt(u1);
    const double b0 = 1.0 - su, b1 = su * (1.0 - u2), b2 = su * u2;
    const d3 q = {(b0 * t[0] + b1 * t[3]) + b2 * t[6], (b0 * t[1] + b1 * t[4]) + b2 * t[7],
                  (b0 * t[2] + b1 * t[5]) + b2 * t[8]};
    const d3 delta = sub(q, p);
    const double dist = norm(delta);
    const double safe = fmax(dist, 1e-12);
    ShadowRay r;
    r.dir = {delta.x / safe, delta.y / safe, delta.z / safe};
    r.tmax = dist * (1.0 - 1e-4);
    r.idx = idx;
    r.su = su;
    r.u2 = u2;
    return r;
}

HRT_DEV ShadowRay shadow_ray(const DevScene& sc, d3 p, uint64_t seed, int64_t pix, int64_t smp,
                             int64_t bounce, int64_t lane) {
    return shadow_ray_h(sc, p, rng::prefix(seed, pix, smp, bounce), lane);
}

// 0 if the sampled emitter point is visible from p, else 1 + emitter index.
HRT_DEV int32_t shadow_code(const DevScene& sc, d3 p, uint64_t seed, int64_t pix, int64_t smp,
                            int64_t bounce, int64_t lane) {
    if (sc.em.n == 0) return 0;
    const ShadowRay r = shadow_ray(sc, p, seed, pix, smp, bounce, lane);
    const bool blocked = bvh::occluded(sc.blockers, p, r.dir, sc.spawn_eps, r.tmax);
    return blocked ? r.idx + 1 : 0;
}

// Mask value of a shadow code: 1, or clip(1 - r_src, 0.02, 1) when blocked.
HRT_DEV double mask_of(const DevScene& sc, int32_t code) {
    if (code == 0) return 1.0;
    return fmin(fmax(1.0 - sc.em.r_src[code - 1], 0.02), 1.0);
}

HRT_DEV double shadow_mask(const DevScene& sc, d3 p, uint64_t seed, int64_t pix, int64_t smp,
                           int64_t bounce, int64_t lane) {
    return mask_of(sc, shadow_code(sc, p, seed, pix, smp, bounce, lane));
}

// ------------------------------------------------------------------ BSDFs
// surface.py:94-95
HRT_DEV d3 reflect(d3 wo, d3 n) {
    const double s = 2.0 * dot(wo, n);
    return {s * n.x - wo.x, s * n.y - wo.y, s * n.z - wo.z};
}

// surface.py:74-91 (_onb + cosine_sample_batch)
HRT_DEV d3 cosine_sample(d3 n, double u1, double u2) {
    const d3 a = fabs(n.x) > 0.9 ? mk(0.0, 1.0, 0.0) : mk(1.0, 0.0, 0.0);
    d3 t = cross(a, n);
    const double tl = norm(t);
    t = {t.x / tl, t.y / tl, t.z / tl};
    const d3 b = cross(n, t);
    const double phi = 6.283185307179586 * u1;
    const double sin_t = sqrt(u2), z = sqrt(1.0 - u2);
    const double lx = cos(phi) * sin_t, ly = sin(phi) * sin_t;
    return {(lx * t.x + ly * b.x) + z * n.x, (lx * t.y + ly * b.y) + z * n.y,
            (lx * t.z + ly * b.z) + z * n.z};
}

// surface.py:102-121 (dielectric_sample_batch)
HRT_DEV d3 dielectric_sample(d3 wo, d3 n, bool front, double ior, double r0, double u) {
    const double cos_i = fmin(fmax(dot(wo, n), 0.0), 1.0);
    const double eta = front ? 1.0 / ior : ior;
    const double sin2_t = eta * eta * fmax(1.0 - cos_i * cos_i, 0.0);
    const bool tir = sin2_t > 1.0;
    const double p_refl = r0 + (1.0 - r0) * pow(1.0 - cos_i, 5.0);
    if (tir || u < p_refl) return reflect(wo, n);
    const double cos_t = sqrt(fmax(1.0 - sin2_t, 0.0));
    const double k = eta * cos_i - cos_t;
    d3 r = {eta * (-wo.x) + k * n.x, eta * (-wo.y) + k * n.y, eta * (-wo.z) + k * n.z};
    const double rn = norm(r);
    const double div = rn > 0 ? rn : 1.0;
    return {r.x / div, r.y / div, r.z / div};
}

}  // namespace path
