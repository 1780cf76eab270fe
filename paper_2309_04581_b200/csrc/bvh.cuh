// bvh.cuh - K2/K3: closest-hit and any-hit BVH traversal.
//
// Hit contract of reference surface.py:377-503: strictly nearest t in
// (t_min, t_max], ties to the smaller global face id, identical to brute
// force. The BVH is the library's own (host SAH build, bvh_build.cpp); node
// boxes are float64 and padded outward on the host so that Moller-Trumbore's
// barycentric tolerance (hits up to 1e-7 outside a face) can never be culled.
// The ray/triangle test is surface.py:243-275 in the same float64 operation
// order (the file is built with --fmad=false), so face ids are bit-exact.
#pragma once
#include "common.cuh"

namespace bvh {

constexpr double BARY_EPS = 1e-7;
constexpr double DET_EPS = 1e-12;
constexpr int kStack = 80;   // binary: <= 1 push per level; tree depth <= 32 + log2(faces) (+ log2(meshes) for a forest)
constexpr int kStackQ = 128; // 4-wide: <= 3 pushes per level over <= ceil(depth / 2) levels

// Reference surface.py:243-275 for one (ray, face) pair; +inf if rejected.
HRT_DEV double moller_trumbore(d3 o, d3 d, const double* __restrict__ t9, double t_min,
                               double t_max) {
    const double ax = t9[3], ay = t9[4], az = t9[5];     // e1
    const double bx = t9[6], by = t9[7], bz = t9[8];     // e2
    const double px = d.y * bz - d.z * by;
    const double py = d.z * bx - d.x * bz;
    const double pz = d.x * by - d.y * bx;
    const double det = (ax * px + ay * py) + az * pz;
    const bool good = fabs(det) > DET_EPS;
    const double inv = 1.0 / (good ? det : 1.0);
    const double sx = o.x - t9[0], sy = o.y - t9[1], sz = o.z - t9[2];
    const double u = ((sx * px + sy * py) + sz * pz) * inv;
    const double qx = sy * az - sz * ay;
    const double qy = sz * ax - sx * az;
    const double qz = sx * ay - sy * ax;
    const double v = ((d.x * qx + d.y * qy) + d.z * qz) * inv;
    const double t = ((bx * qx + by * qy) + bz * qz) * inv;
    const bool ok = good && (u >= -BARY_EPS) && (v >= -BARY_EPS) && (u + v <= 1.0 + BARY_EPS) &&
                    (t > t_min) && (t <= t_max);
    return ok ? t : INFINITY;
}

struct RayInv {
    d3 o;
    double ix, iy, iz;
};

HRT_DEV RayInv prep(d3 o, d3 d) { return {o, 1.0 / d.x, 1.0 / d.y, 1.0 / d.z}; }

// Slab overlap of a node with [t0, t1]; NaN (0 * inf on an axis-aligned ray
// touching a slab plane) widens to the whole axis as surface.py:412-420 does.
HRT_DEV bool node_hit(const BvhNode& n, const RayInv& r, double t0, double t1, double& near) {
    double ta = (n.lo[0] - r.o.x) * r.ix, tb = (n.hi[0] - r.o.x) * r.ix;
    double lo = (ta != ta || tb != tb) ? -INFINITY : fmin(ta, tb);
    double hi = (ta != ta || tb != tb) ? INFINITY : fmax(ta, tb);
    ta = (n.lo[1] - r.o.y) * r.iy; tb = (n.hi[1] - r.o.y) * r.iy;
    lo = fmax(lo, (ta != ta || tb != tb) ? -INFINITY : fmin(ta, tb));
    hi = fmin(hi, (ta != ta || tb != tb) ? INFINITY : fmax(ta, tb));
    ta = (n.lo[2] - r.o.z) * r.iz; tb = (n.hi[2] - r.o.z) * r.iz;
    lo = fmax(lo, (ta != ta || tb != tb) ? -INFINITY : fmin(ta, tb));
    hi = fmin(hi, (ta != ta || tb != tb) ? INFINITY : fmax(ta, tb));
    near = fmax(lo, t0);
    return near <= fmin(hi, t1);
}

// Nearest hit; returns global face id or -1, t in `best_t`.
HRT_DEV int32_t closest(const DevBvh& b, d3 o, d3 d, double t_min, double t_max, double& best_t) {
    best_t = INFINITY;
    int32_t best_f = -1;
    if (b.n_faces == 0) return -1;
    const RayInv r = prep(o, d);
    int32_t stack[kStack];
    int sp = 0;
    int32_t node = 0;
    double nr;
    if (!node_hit(b.nodes[0], r, t_min, t_max, nr)) return -1;
    while (true) {
        const BvhNode n = b.nodes[node];
        if (n.count > 0) {
            for (int i = 0; i < n.count; ++i) {
                const int32_t li = n.first + i;
                const double t = moller_trumbore(o, d, b.tri + 9 * (size_t)li, t_min, t_max);
                if (t < INFINITY) {
                    const int32_t f = b.tri_id[li];
                    if (t < best_t || (t == best_t && f < best_f)) { best_t = t; best_f = f; }
                }
            }
        } else {
            const double lim = fmin(t_max, best_t);
            double n0, n1;
            const bool h0 = node_hit(b.nodes[n.first], r, t_min, lim, n0);
            const bool h1 = node_hit(b.nodes[n.first + 1], r, t_min, lim, n1);
            if (h0 && h1) {
                const bool first0 = n0 <= n1;
                if (sp < kStack) stack[sp++] = first0 ? n.first + 1 : n.first;
                node = first0 ? n.first : n.first + 1;
                continue;
            }
            if (h0 || h1) { node = h0 ? n.first : n.first + 1; continue; }
        }
        // pop, skipping nodes that can no longer hold a hit <= best_t
        bool found = false;
        while (sp > 0) {
            const int32_t c = stack[--sp];
            if (node_hit(b.nodes[c], r, t_min, fmin(t_max, best_t), nr)) { node = c; found = true; break; }
        }
        if (!found) break;
    }
    return best_f;
}

// True if any face lies in (t_min, t_max] (reference surface.py:442-478).
HRT_DEV bool any_hit(const DevBvh& b, d3 o, d3 d, double t_min, double t_max) {
    if (b.n_faces == 0) return false;
    const RayInv r = prep(o, d);
    int32_t stack[kStack];
    int sp = 0;
    int32_t node = 0;
    double nr;
    if (!node_hit(b.nodes[0], r, t_min, t_max, nr)) return false;
    while (true) {
        const BvhNode n = b.nodes[node];
        if (n.count > 0) {
            for (int i = 0; i < n.count; ++i) {
                if (moller_trumbore(o, d, b.tri + 9 * (size_t)(n.first + i), t_min, t_max) < INFINITY)
                    return true;
            }
        } else {
            double n0, n1;
            const bool h0 = node_hit(b.nodes[n.first], r, t_min, t_max, n0);
            const bool h1 = node_hit(b.nodes[n.first + 1], r, t_min, t_max, n1);
            if (h0 && h1) {
                if (sp < kStack) stack[sp++] = n.first + 1;
                node = n.first;
                continue;
            }
            if (h0 || h1) { node = h0 ? n.first : n.first + 1; continue; }
        }
        if (sp == 0) break;
        node = stack[--sp];
    }
    return false;
}

// ------------------------------------------- float32-culled traversal
// Box tests run in float32 on WNode (half the bytes of the float64 tree,
// both children per 64-byte load); they only cull, never decide: the boxes
// are rounded outward and padded by 1e-5 * max(1, |coord|), the ray
// interval is widened by 1e-5 relative + absolute, so every box the exact
// test would enter is entered here, and every candidate triangle goes
// through the float64 Moller-Trumbore above. Hits are therefore the
// reference's (nearest t, ties to the smaller face id) bit for bit.
struct Ray32 {
    float ox, oy, oz, ix, iy, iz;
};

// Reciprocal direction with |d| < 1e-30 (zero included) taken as +-1e-30:
// the slab products then never form 0 * inf = NaN, so the box test needs no
// NaN handling. Still conservative: such a ray parallel to a slab gets an
// interval of +-1e30-scale t (the whole axis when its origin is inside the
// slab, far outside the scene when it is not), as the exact reciprocal would.
HRT_DEV float rcp_safe(double dd) {
    const float f = (float)dd;
    return 1.0f / (fabsf(f) < 1e-30f ? copysignf(1e-30f, f) : f);
}

HRT_DEV Ray32 prep32(d3 o, d3 d) {
    Ray32 r;
    r.ox = (float)o.x; r.oy = (float)o.y; r.oz = (float)o.z;
    r.ix = rcp_safe(d.x); r.iy = rcp_safe(d.y); r.iz = rcp_safe(d.z);
    return r;
}

HRT_DEV float t_lo32(double t) { return t <= 0.0 ? (float)t * 1.00001f - 1e-5f : (float)t * 0.99999f - 1e-5f; }
HRT_DEV float t_hi32(double t) { return (float)t * 1.00001f + 1e-5f; }

HRT_DEV void slab_axis(float lo, float hi, float o, float inv, float& tn, float& tf) {
    const float ta = (lo - o) * inv, tb = (hi - o) * inv;     // finite inv: no NaN (rcp_safe)
    tn = fmaxf(tn, fminf(ta, tb));
    tf = fminf(tf, fmaxf(ta, tb));
}

HRT_DEV bool box32(float lx, float ly, float lz, float hx, float hy, float hz, const Ray32& r,
                   float t0, float t1, float& near) {
    float tn = t0, tf = t1;
    slab_axis(lx, hx, r.ox, r.ix, tn, tf);
    slab_axis(ly, hy, r.oy, r.iy, tn, tf);
    slab_axis(lz, hz, r.oz, r.iz, tn, tf);
    near = tn;
    return tn <= tf;
}

HRT_DEV void wchildren(const WNode& w, const Ray32& r, float t0, float t1, bool& h0, bool& h1,
                       float& n0, float& n1) {
    h0 = box32(w.a.x, w.a.y, w.a.z, w.a.w, w.b.x, w.b.y, r, t0, t1, n0);
    h1 = box32(w.b.z, w.b.w, w.c.x, w.c.y, w.c.z, w.c.w, r, t0, t1, n1);
}

HRT_DEV WNode load_w(const WNode* __restrict__ nodes, int32_t i) {
    const float4* p = reinterpret_cast<const float4*>(nodes + i);
    WNode w;
    w.a = __ldg(p);
    w.b = __ldg(p + 1);
    w.c = __ldg(p + 2);
    w.r = __ldg(reinterpret_cast<const int4*>(p + 3));
    return w;
}

// Leaf of ref (< 0): nearest-hit update over its triangles.
HRT_DEV void leaf_closest(const DevBvh& b, int32_t ref, d3 o, d3 d, double t_min, double t_max,
                          double& best_t, int32_t& best_f) {
    const int32_t code = ~ref, first = code >> 3, count = code & 7;
    for (int i = 0; i < count; ++i) {
        const int32_t li = first + i;
        const double t = moller_trumbore(o, d, b.tri + 9 * (size_t)li, t_min, t_max);
        if (t < INFINITY) {
            const int32_t f = b.tri_id[li];
            if (t < best_t || (t == best_t && f < best_f)) { best_t = t; best_f = f; }
        }
    }
}

HRT_DEV bool leaf_any(const DevBvh& b, int32_t ref, d3 o, d3 d, double t_min, double t_max) {
    const int32_t code = ~ref, first = code >> 3, count = code & 7;
    for (int i = 0; i < count; ++i)
        if (moller_trumbore(o, d, b.tri + 9 * (size_t)(first + i), t_min, t_max) < INFINITY) return true;
    return false;
}

// Nearest hit (surface.py:377-440 contract); global face id or -1.
HRT_DEV int32_t closest_w(const DevBvh& b, d3 o, d3 d, double t_min, double t_max, double& best_t) {
    best_t = INFINITY;
    int32_t best_f = -1;
    if (b.n_faces == 0) return -1;
    const Ray32 r = prep32(o, d);
    const float t0 = t_lo32(t_min);
    int32_t stack[kStack];
    float stack_t[kStack];
    int sp = 0;
    int32_t cur = 0;
    while (true) {
        const WNode w = load_w(b.wnodes, cur);
        const float t1 = t_hi32(fmin(t_max, best_t));
        bool h0, h1;
        float n0, n1;
        wchildren(w, r, t0, t1, h0, h1, n0, n1);
        if (h0 && w.r.x < 0) { leaf_closest(b, w.r.x, o, d, t_min, t_max, best_t, best_f); h0 = false; }
        if (h1 && w.r.y < 0) { leaf_closest(b, w.r.y, o, d, t_min, t_max, best_t, best_f); h1 = false; }
        if (h0 && h1) {
            const bool first0 = n0 <= n1;
            if (sp < kStack) {
                stack[sp] = first0 ? w.r.y : w.r.x;
                stack_t[sp] = first0 ? n1 : n0;
                ++sp;
            }
            cur = first0 ? w.r.x : w.r.y;
            continue;
        }
        if (h0 || h1) { cur = h0 ? w.r.x : w.r.y; continue; }
        // pop, skipping subtrees whose entry lies beyond the current best hit
        bool found = false;
        const float lim = t_hi32(fmin(t_max, best_t));
        while (sp > 0) {
            --sp;
            if (stack_t[sp] <= lim) { cur = stack[sp]; found = true; break; }
        }
        if (!found) break;
    }
    return best_f;
}

// Can the segment reach any box of the tree at all? (root WNode's children)
HRT_DEV bool root_overlap(const DevBvh& b, d3 o, d3 d, double t_min, double t_max) {
    if (b.n_faces == 0) return false;
    const Ray32 r = prep32(o, d);
    const WNode w = load_w(b.wnodes, 0);
    bool h0, h1;
    float n0, n1;
    wchildren(w, r, t_lo32(t_min), t_hi32(t_max), h0, h1, n0, n1);
    return h0 || h1;
}

// True if any face lies in (t_min, t_max] (surface.py:442-478).
HRT_DEV bool any_hit_w(const DevBvh& b, d3 o, d3 d, double t_min, double t_max) {
    if (b.n_faces == 0) return false;
    const Ray32 r = prep32(o, d);
    const float t0 = t_lo32(t_min), t1 = t_hi32(t_max);
    int32_t stack[kStack];
    int sp = 0;
    int32_t cur = 0;
    while (true) {
        const WNode w = load_w(b.wnodes, cur);
        bool h0, h1;
        float n0, n1;
        wchildren(w, r, t0, t1, h0, h1, n0, n1);
        if (h0 && w.r.x < 0) {
            if (leaf_any(b, w.r.x, o, d, t_min, t_max)) return true;
            h0 = false;
        }
        if (h1 && w.r.y < 0) {
            if (leaf_any(b, w.r.y, o, d, t_min, t_max)) return true;
            h1 = false;
        }
        if (h0 && h1) {                  // nearer child first: occluders are found sooner
            const bool near0 = n0 <= n1;
            if (sp < kStack) stack[sp++] = near0 ? w.r.y : w.r.x;
            cur = near0 ? w.r.x : w.r.y;
            continue;
        }
        if (h0 || h1) { cur = h0 ? w.r.x : w.r.y; continue; }
        if (sp == 0) break;
        cur = stack[--sp];
    }
    return false;
}

// ---------------------------------------------------- 4-wide traversal
// Any-hit traversals fetch the node's refs and lo.x box row through the LSU
// path and the other five box rows through the TEX path (a float4 texture
// over the same array, same bits), so divergent traversals spread their node
// fetches over both L1TEX data pipes (round-1 ncu of the shadow tracer: LSU
// data pipe 84 % busy; hi rows on TEX: shadow stage -4 %; round 2, session 2:
// lo.y and lo.z on TEX too, with LSU still at 73 %: cfg4 shadow stage
// 664 -> 641 ms; all six: 650 ms). Closest-hit traversals keep LSU only
// (+4 % with the split).
#ifndef HRT_QNODE_TEX
#define HRT_QNODE_TEX 1
#endif
#ifndef HRT_QNODE_TEX_FIELDS
#define HRT_QNODE_TEX_FIELDS 5      // box float4s (from the end: hiz, hiy, hix, loz, loy, lox) fetched through TEX
#endif
template <bool kTex = false>
HRT_DEV QNode load_q(const DevBvh& b, int32_t i) {
    const float4* p = reinterpret_cast<const float4*>(b.qnodes + i);
    QNode q;
    if (kTex && HRT_QNODE_TEX && b.qtex) {
        const int t = 8 * i;
        constexpr int NT = HRT_QNODE_TEX_FIELDS;
        q.lox = NT >= 6 ? tex1Dfetch<float4>(b.qtex, t) : __ldg(p);
        q.loy = NT >= 5 ? tex1Dfetch<float4>(b.qtex, t + 1) : __ldg(p + 1);
        q.loz = NT >= 4 ? tex1Dfetch<float4>(b.qtex, t + 2) : __ldg(p + 2);
        q.hix = NT >= 3 ? tex1Dfetch<float4>(b.qtex, t + 3) : __ldg(p + 3);
        q.hiy = NT >= 2 ? tex1Dfetch<float4>(b.qtex, t + 4) : __ldg(p + 4);
        q.hiz = NT >= 1 ? tex1Dfetch<float4>(b.qtex, t + 5) : __ldg(p + 5);
    } else {
        q.lox = __ldg(p); q.loy = __ldg(p + 1); q.loz = __ldg(p + 2);
        q.hix = __ldg(p + 3); q.hiy = __ldg(p + 4); q.hiz = __ldg(p + 5);
    }
    q.ref = __ldg(reinterpret_cast<const int4*>(p + 6));
    return q;
}

// Box tests of the 4 children; hit mask bit k, entry distance near[k].
HRT_DEV uint32_t qchildren(const QNode& q, const Ray32& r, float t0, float t1, float near[4]) {
    uint32_t m = 0;
    const float lx[4] = {q.lox.x, q.lox.y, q.lox.z, q.lox.w}, ly[4] = {q.loy.x, q.loy.y, q.loy.z, q.loy.w};
    const float lz[4] = {q.loz.x, q.loz.y, q.loz.z, q.loz.w}, hx[4] = {q.hix.x, q.hix.y, q.hix.z, q.hix.w};
    const float hy[4] = {q.hiy.x, q.hiy.y, q.hiy.z, q.hiy.w}, hz[4] = {q.hiz.x, q.hiz.y, q.hiz.z, q.hiz.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (box32(lx[k], ly[k], lz[k], hx[k], hy[k], hz[k], r, t0, t1, near[k])) m |= 1u << k;
    return m;
}

HRT_DEV int32_t qref(const QNode& q, int k) {
    return k == 0 ? q.ref.x : (k == 1 ? q.ref.y : (k == 2 ? q.ref.z : q.ref.w));
}

// Nearest hit on the 4-wide tree (surface.py:377-440 contract).
HRT_DEV int32_t closest_q(const DevBvh& b, d3 o, d3 d, double t_min, double t_max, double& best_t) {
    best_t = INFINITY;
    int32_t best_f = -1;
    if (b.n_faces == 0) return -1;
    const Ray32 r = prep32(o, d);
    const float t0 = t_lo32(t_min);
    int32_t stack[kStackQ];
    float stack_t[kStackQ];
    int sp = 0;
    int32_t cur = 0;
    float lim = t_hi32(t_max);        // t_hi32(min(t_max, best_t)), refreshed when a leaf hits
    while (true) {
        const QNode q = load_q(b, cur);
        float nr[4];
        uint32_t m = qchildren(q, r, t0, lim, nr);
        // leaves first (they can only shrink best_t)
        const uint32_t leaves = m & ((qref(q, 0) < 0 ? 1u : 0u) | (qref(q, 1) < 0 ? 2u : 0u) |
                                     (qref(q, 2) < 0 ? 4u : 0u) | (qref(q, 3) < 0 ? 8u : 0u));
        if (leaves) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (leaves >> k & 1u) leaf_closest(b, qref(q, k), o, d, t_min, t_max, best_t, best_f);
            m &= ~leaves;
            lim = t_hi32(fmin(t_max, best_t));
        }
        // inner children: nearest next, the rest pushed far-to-near
        int32_t next = -1;
        while (m) {
            int kb = -1;
            float tb = -INFINITY;
#pragma unroll
            for (int k = 0; k < 4; ++k)              // farthest remaining first onto the stack
                if ((m >> k & 1u) && nr[k] >= tb) { tb = nr[k]; kb = k; }
            m &= ~(1u << kb);
            if (tb > lim) continue;
            if (m == 0) { next = qref(q, kb); break; }
            if (sp < kStackQ) { stack[sp] = qref(q, kb); stack_t[sp] = tb; ++sp; }
        }
        if (next >= 0) { cur = next; continue; }
        bool found = false;
        while (sp > 0) {
            --sp;
            if (stack_t[sp] <= lim) { cur = stack[sp]; found = true; break; }
        }
        if (!found) break;
    }
    return best_f;
}

// Nearest hit with 4 lanes per ray (a group of 4 consecutive lanes, gl = lane
// in group): lane k tests child k of the current node - its box and, for a
// leaf child, its triangles - and the group combines the results by shuffles.
// For the latency-bound case (few rays, long traversals): a node visit costs
// one box test and one leaf test instead of four of each. Every lane keeps
// the same traversal state. The answer is the lexicographic minimum (t, face)
// over the triangles whose boxes the ray reaches, as closest_q's.
HRT_DEV int32_t closest_q_coop(const DevBvh& b, d3 o, d3 d, double t_min, double t_max, double& best_t,
                               uint32_t gmask, uint32_t gbase, uint32_t gl) {
    best_t = INFINITY;
    int32_t best_f = -1;
    if (b.n_faces == 0) return -1;
    const Ray32 r = prep32(o, d);
    const float t0 = t_lo32(t_min);
    float lim = t_hi32(t_max);
    int32_t stack[kStackQ];
    float stack_t[kStackQ];
    int sp = 0;
    int32_t cur = 0;
    while (true) {
        const float* q = reinterpret_cast<const float*>(b.qnodes + cur);
        const float lx = __ldg(q + gl), ly = __ldg(q + 4 + gl), lz = __ldg(q + 8 + gl);
        const float hx = __ldg(q + 12 + gl), hy = __ldg(q + 16 + gl), hz = __ldg(q + 20 + gl);
        const int32_t ref = __ldg(reinterpret_cast<const int32_t*>(q) + 24 + gl);
        float nr;
        const bool hit = box32(lx, ly, lz, hx, hy, hz, r, t0, lim, nr);
        // leaf child of this lane
        double lt = INFINITY;
        int32_t lf = 0x7fffffff;
        if (hit && ref < 0) {
            const int32_t code = ~ref, first = code >> 3, count = code & 7;
            for (int i = 0; i < count; ++i) {
                const int32_t li = first + i;
                const double t = moller_trumbore(o, d, b.tri + 9 * (size_t)li, t_min, t_max);
                if (t < INFINITY) {
                    const int32_t f = b.tri_id[li];
                    if (t < lt || (t == lt && f < lf)) { lt = t; lf = f; }
                }
            }
        }
        const uint32_t leaves = (__ballot_sync(gmask, hit && ref < 0) >> gbase) & 0xFu;
        if (leaves) {
#pragma unroll
            for (int off = 1; off < 4; off <<= 1) {
                const double ot = __shfl_xor_sync(gmask, lt, off);
                const int32_t of = __shfl_xor_sync(gmask, lf, off);
                if (ot < lt || (ot == lt && of < lf)) { lt = ot; lf = of; }
            }
            if (lt < best_t || (lt == best_t && lf < best_f)) { best_t = lt; best_f = lf; }
            lim = t_hi32(fmin(t_max, best_t));
        }
        // inner children: nearest next, the rest pushed far-to-near (as closest_q)
        uint32_t m = (__ballot_sync(gmask, hit && ref >= 0) >> gbase) & 0xFu;
        float nr4[4];
        int32_t ref4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            nr4[k] = __shfl_sync(gmask, nr, (int)(gbase + k));
            ref4[k] = __shfl_sync(gmask, ref, (int)(gbase + k));
        }
        int32_t next = -1;
        while (m) {
            int kb = -1;
            float tb = -INFINITY;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if ((m >> k & 1u) && nr4[k] >= tb) { tb = nr4[k]; kb = k; }
            m &= ~(1u << kb);
            if (tb > lim) continue;
            if (m == 0) { next = ref4[kb]; break; }
            if (sp < kStackQ) { stack[sp] = ref4[kb]; stack_t[sp] = tb; ++sp; }
        }
        if (next >= 0) { cur = next; continue; }
        bool found = false;
        while (sp > 0) {
            --sp;
            if (stack_t[sp] <= lim) { cur = stack[sp]; found = true; break; }
        }
        if (!found) break;
    }
    return best_f;
}

// True if any face lies in (t_min, t_max] (surface.py:442-478), 4-wide tree.
HRT_DEV bool any_hit_q(const DevBvh& b, d3 o, d3 d, double t_min, double t_max) {
    if (b.n_faces == 0) return false;
    const Ray32 r = prep32(o, d);
    const float t0 = t_lo32(t_min), t1 = t_hi32(t_max);
    int32_t stack[kStackQ];
    int sp = 0;
    int32_t cur = 0;
    while (true) {
        const QNode q = load_q<true>(b, cur);
        float nr[4];
        uint32_t m = qchildren(q, r, t0, t1, nr);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((m >> k & 1u) && qref(q, k) < 0) {
                if (leaf_any(b, qref(q, k), o, d, t_min, t_max)) return true;
                m &= ~(1u << k);
            }
        int32_t next = -1;
        while (m) {
            int kb = -1;
            float tb = -INFINITY;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if ((m >> k & 1u) && nr[k] >= tb) { tb = nr[k]; kb = k; }
            m &= ~(1u << kb);
            if (m == 0) { next = qref(q, kb); break; }
            if (sp < kStackQ) stack[sp++] = qref(q, kb);
        }
        if (next >= 0) { cur = next; continue; }
        if (sp == 0) break;
        cur = stack[--sp];
    }
    return false;
}

#ifndef HRT_BVH64
#define HRT_BVH64 0      // 1: traverse the float64 tree (reference-order culling)
#endif
#ifndef HRT_BVH_WIDTH
#define HRT_BVH_WIDTH 4  // traversal tree: 4-wide QNodes (2: the binary WNode tree)
#endif
HRT_DEV int32_t nearest(const DevBvh& b, d3 o, d3 d, double t_min, double t_max, double& best_t) {
    if (HRT_BVH64) return closest(b, o, d, t_min, t_max, best_t);
    return HRT_BVH_WIDTH == 4 ? closest_q(b, o, d, t_min, t_max, best_t) : closest_w(b, o, d, t_min, t_max, best_t);
}
HRT_DEV bool occluded(const DevBvh& b, d3 o, d3 d, double t_min, double t_max) {
    if (HRT_BVH64) return any_hit(b, o, d, t_min, t_max);
    return HRT_BVH_WIDTH == 4 ? any_hit_q(b, o, d, t_min, t_max) : any_hit_w(b, o, d, t_min, t_max);
}

// WNode child boxes from the float64 tree after a refit (src: float64 node
// index per child slot, -1 = empty). Same rounding as the host (hrt.cu wbox).
HRT_DEV void wbox_dev(const BvhNode& n, float lo[3], float hi[3]) {
    double mag = 1.0;
    for (int a = 0; a < 3; ++a) mag = fmax(mag, fmax(fabs(n.lo[a]), fabs(n.hi[a])));
    const double pad = 1e-5 * mag;
    for (int a = 0; a < 3; ++a) {
        lo[a] = __double2float_rd(n.lo[a] - pad);
        hi[a] = __double2float_ru(n.hi[a] + pad);
    }
}

__global__ void k_wsync(WNode* w, const int2* __restrict__ src, const BvhNode* __restrict__ nodes,
                        int32_t begin, int32_t n) {
    for (int32_t i = begin + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int2 sidx = src[i];
        float l0[3], h0[3], l1[3], h1[3];
        if (sidx.x >= 0) wbox_dev(nodes[sidx.x], l0, h0);
        else { l0[0] = l0[1] = l0[2] = h0[0] = h0[1] = h0[2] = 1e30f; }
        if (sidx.y >= 0) wbox_dev(nodes[sidx.y], l1, h1);
        else { l1[0] = l1[1] = l1[2] = h1[0] = h1[1] = h1[2] = 1e30f; }
        w[i].a = make_float4(l0[0], l0[1], l0[2], h0[0]);
        w[i].b = make_float4(h0[1], h0[2], l1[0], l1[1]);
        w[i].c = make_float4(l1[2], h1[0], h1[1], h1[2]);
    }
}

// ------------------------------------------------------------ GPU refit (K11)
// Moving meshes keep their topology; the tree is refit bottom-up: each leaf
// rebuilds its padded box from its (new) triangles, then climbs; at every
// inner node the second child to arrive (arrival counter) forms the union.
// Boxes use the host builder's padding rule (bvh_build.cpp face_box), so
// hits stay exactly those of brute force.
HRT_DEV void face_box_pad(const double* t9, double lo[3], double hi[3]) {
    double ext = 0.0, mag = 1.0;
    for (int a = 0; a < 3; ++a) {
        const double v0 = t9[a], v1 = t9[a] + t9[3 + a], v2 = t9[a] + t9[6 + a];
        lo[a] = fmin(v0, fmin(v1, v2));
        hi[a] = fmax(v0, fmax(v1, v2));
        ext = fmax(ext, hi[a] - lo[a]);
        mag = fmax(mag, fmax(fabs(lo[a]), fabs(hi[a])));
    }
    const double pad = 1e-6 * ext + 1e-12 * mag;
    for (int a = 0; a < 3; ++a) { lo[a] -= pad; hi[a] += pad; }
}

__global__ void k_permute_tris(const double* __restrict__ v0, const double* __restrict__ e1,
                               const double* __restrict__ e2, const int32_t* __restrict__ tri_id,
                               int32_t n, double* tri) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int32_t f = tri_id[i];
        for (int a = 0; a < 3; ++a) {
            tri[9 * (size_t)i + a] = v0[3 * (size_t)f + a];
            tri[9 * (size_t)i + 3 + a] = e1[3 * (size_t)f + a];
            tri[9 * (size_t)i + 6 + a] = e2[3 * (size_t)f + a];
        }
    }
}

__global__ void k_refit(BvhNode* nodes, const int32_t* __restrict__ parent,
                        const int32_t* __restrict__ leaves, int32_t n_leaves, const double* tri,
                        int32_t* visits) {
    for (int32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < n_leaves;
         li += gridDim.x * blockDim.x) {
        int32_t node = leaves[li];
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        const BvhNode leaf = nodes[node];
        for (int i = 0; i < leaf.count; ++i) {
            double a[3], b[3];
            face_box_pad(tri + 9 * (size_t)(leaf.first + i), a, b);
            for (int k = 0; k < 3; ++k) { lo[k] = fmin(lo[k], a[k]); hi[k] = fmax(hi[k], b[k]); }
        }
        for (int k = 0; k < 3; ++k) { nodes[node].lo[k] = lo[k]; nodes[node].hi[k] = hi[k]; }
        while (true) {
            const int32_t p = parent[node];
            if (p < 0) break;
            __threadfence();
            if (atomicAdd(&visits[p], 1) == 0) break;      // sibling not done yet
            __threadfence();
            const int32_t c = nodes[p].first;
            for (int k = 0; k < 3; ++k) {
                const double l0 = __ldcg(&nodes[c].lo[k]), l1 = __ldcg(&nodes[c + 1].lo[k]);
                const double h0 = __ldcg(&nodes[c].hi[k]), h1 = __ldcg(&nodes[c + 1].hi[k]);
                nodes[p].lo[k] = fmin(l0, l1);
                nodes[p].hi[k] = fmax(h0, h1);
            }
            node = p;
        }
    }
}


// Root boxes of a forest's trees (6 doubles each) for the host top-level build.
__global__ void k_root_boxes(const BvhNode* __restrict__ nodes, const int32_t* __restrict__ roots, int32_t g,
                             double* out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g) return;
    const BvhNode& n = nodes[roots[i]];
    for (int a = 0; a < 3; ++a) {
        out[6 * i + a] = n.lo[a];
        out[6 * i + 3 + a] = n.hi[a];
    }
}

// Rigid per-mesh motion on the device (cfg3): world corner = M * p with
// M the mesh's 3x4 world_from_object, row r as ((m0*x + m1*y) + m2*z) + m3
// (no FMA; paper_2309_04581_b200.configs.apply_rigid is the same order),
// then v0 | e1 = w1 - w0 | e2 = w2 - w0 into the refit staging buffer and the
// unit normal of face_normals_of (surface.py:169-176 order).
__global__ void k_rigid_faces(const double* __restrict__ base, const int32_t* __restrict__ mesh_of,
                              const double* __restrict__ xf, int32_t n_meshes, int32_t n, double* src,
                              double* normal) {
    const size_t n3 = 3 * (size_t)n;
    for (int32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
        const int32_t mi = min(mesh_of[f], n_meshes - 1);
        const double* m = xf + 12 * (size_t)mi;
        double w[3][3];
        for (int c = 0; c < 3; ++c) {
            const double* p = base + 9 * (size_t)f + 3 * c;
            for (int r = 0; r < 3; ++r)
                w[c][r] = ((m[4 * r] * p[0] + m[4 * r + 1] * p[1]) + m[4 * r + 2] * p[2]) + m[4 * r + 3];
        }
        double e1[3], e2[3];
        for (int r = 0; r < 3; ++r) {
            e1[r] = w[1][r] - w[0][r];
            e2[r] = w[2][r] - w[0][r];
            src[3 * (size_t)f + r] = w[0][r];
            src[n3 + 3 * (size_t)f + r] = e1[r];
            src[2 * n3 + 3 * (size_t)f + r] = e2[r];
        }
        const double nx = e1[1] * e2[2] - e1[2] * e2[1];
        const double ny = e1[2] * e2[0] - e1[0] * e2[2];
        const double nz = e1[0] * e2[1] - e1[1] * e2[0];
        const double len = sqrt((nx * nx + ny * ny) + nz * nz);
        normal[3 * (size_t)f] = nx / len;
        normal[3 * (size_t)f + 1] = ny / len;
        normal[3 * (size_t)f + 2] = nz / len;
    }
}

// Blocker staging from the main one (blocker face i = global face map[i]).
__global__ void k_gather_faces(const double* __restrict__ src, int32_t n, const int32_t* __restrict__ map,
                               int32_t nb, double* dst) {
    const size_t n3 = 3 * (size_t)n, b3 = 3 * (size_t)nb;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
        const int32_t f = map[i];
        for (int k = 0; k < 3; ++k)
            for (int r = 0; r < 3; ++r) dst[k * b3 + 3 * (size_t)i + r] = src[k * n3 + 3 * (size_t)f + r];
    }
}

// QNode child boxes from the float64 tree after a refit (src: float64 node per
// slot, -1 = not from the tree: empty slot or a forest top-level slot).
__global__ void k_qsync(QNode* q, const int4* __restrict__ src, const BvhNode* __restrict__ nodes,
                        int32_t begin, int32_t n) {
    for (int32_t i = begin + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int4 sidx = src[i];
        const int32_t si[4] = {sidx.x, sidx.y, sidx.z, sidx.w};
        float lo[4][3], hi[4][3];
        for (int k = 0; k < 4; ++k) {
            if (si[k] >= 0) {
                BvhNode nb = nodes[si[k]];
                wbox_dev(nb, lo[k], hi[k]);
            }
        }
        QNode x = q[i];
        float* f = reinterpret_cast<float*>(&x);       // lox[4] loy[4] loz[4] hix[4] hiy[4] hiz[4]
        for (int k = 0; k < 4; ++k) {
            if (si[k] < 0) continue;
            for (int a = 0; a < 3; ++a) {
                f[4 * a + k] = lo[k][a];
                f[12 + 4 * a + k] = hi[k][a];
            }
        }
        q[i] = x;
    }
}


// ------------------------------------------------- shadow entry table
// Light-space culling of shadow any-hit queries, exact. A shadow ray from a
// point x in world cell C towards a light point q in patch Q of emitter e
// (q is bilinear in (sqrt(u1), u2), so a patch's points lie in the convex
// hull of its 4 corner points) stays inside H = hull(C u Q); a triangle it
// hits meets H, and so does every tree box above that triangle. The entry of
// (C, e, Q) is found from the root by descending while exactly one child box
// can meet H; it is -2 when no child box can meet H (nothing can be hit).
// Separation is shown on 7 axes (x, y, z and four across the beam C -> Q) in
// float64 with H padded: an axis only ever proves a real separation, so a
// traversal started at the entry finds every hit a traversal from the root
// finds (and the blocked / visible answer is identical).
struct Hull {
    d3 ax[7];
    double lo[7], hi[7];
};

HRT_DEV bool hull_apart(const Hull& H, float lx, float ly, float lz, float hx, float hy, float hz) {
    const double cx = 0.5 * ((double)lx + (double)hx), cy = 0.5 * ((double)ly + (double)hy),
                 cz = 0.5 * ((double)lz + (double)hz);
    const double ex = 0.5 * ((double)hx - (double)lx), ey = 0.5 * ((double)hy - (double)ly),
                 ez = 0.5 * ((double)hz - (double)lz);
#pragma unroll
    for (int a = 0; a < 7; ++a) {
        const d3 n = H.ax[a];
        const double c = n.x * cx + n.y * cy + n.z * cz;
        const double r = fabs(n.x) * ex + fabs(n.y) * ey + fabs(n.z) * ez;
        if (c + r < H.lo[a] || c - r > H.hi[a]) return true;
    }
    return false;
}

// entry index -> ((cell * n_emitters + emitter) * P + v) * P + u, cell = (z * g + y) * g + x
__global__ void k_shadow_entry(DevBvh b, DevEmitters em, d3 glo, d3 cell, int32_t g, int32_t P,
                               int32_t* out, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t pu = (int32_t)(e % P), pv = (int32_t)((e / P) % P);
        const int64_t rest = e / ((int64_t)P * P);
        const int32_t emi = (int32_t)(rest % em.n);
        const int64_t c = rest / em.n;
        const int32_t ci[3] = {(int32_t)(c % g), (int32_t)((c / g) % g), (int32_t)(c / ((int64_t)g * g))};
        d3 V[12];
        for (int k = 0; k < 8; ++k)
            V[k] = mk(glo.x + (ci[0] + (k & 1)) * cell.x, glo.y + (ci[1] + ((k >> 1) & 1)) * cell.y,
                      glo.z + (ci[2] + (k >> 2)) * cell.z);
        const double* t = em.tris + 9 * emi;
        for (int k = 0; k < 4; ++k) {
            const double su = (double)(pu + (k & 1)) / P, u2 = (double)(pv + (k >> 1)) / P;
            const double b0 = 1.0 - su, b1 = su * (1.0 - u2), b2 = su * u2;
            V[8 + k] = mk(b0 * t[0] + b1 * t[3] + b2 * t[6], b0 * t[1] + b1 * t[4] + b2 * t[7],
                          b0 * t[2] + b1 * t[5] + b2 * t[8]);
        }
        d3 cc = mk(0, 0, 0), pc = mk(0, 0, 0);
        double big = 1.0;
        for (int k = 0; k < 12; ++k) {
            if (k < 8) cc = add(cc, scale(V[k], 0.125)); else pc = add(pc, scale(V[k], 0.25));
            big = fmax(big, fmax(fabs(V[k].x), fmax(fabs(V[k].y), fabs(V[k].z))));
        }
        const double pad = 1e-6 * big;
        Hull H;
        H.ax[0] = mk(1, 0, 0); H.ax[1] = mk(0, 1, 0); H.ax[2] = mk(0, 0, 1);
        d3 D = sub(pc, cc);
        const double dl = norm(D);
        D = dl > 1e-12 ? scale(D, 1.0 / dl) : mk(1, 0, 0);
        const d3 ek = (fabs(D.x) <= fabs(D.y) && fabs(D.x) <= fabs(D.z)) ? mk(1, 0, 0)
                      : (fabs(D.y) <= fabs(D.z) ? mk(0, 1, 0) : mk(0, 0, 1));
        d3 U = cross(D, ek);
        U = scale(U, 1.0 / norm(U));
        const d3 W = cross(D, U);
        H.ax[3] = U; H.ax[4] = W;
        H.ax[5] = scale(add(U, W), 0.7071067811865476);
        H.ax[6] = scale(sub(U, W), 0.7071067811865476);
        for (int a = 0; a < 7; ++a) {
            double lo = INFINITY, hi = -INFINITY;
            for (int k = 0; k < 12; ++k) {
                const double v = dot(H.ax[a], V[k]);
                lo = fmin(lo, v);
                hi = fmax(hi, v);
            }
            const double w = pad * (fabs(H.ax[a].x) + fabs(H.ax[a].y) + fabs(H.ax[a].z)) + 1e-12 * big;
            H.lo[a] = lo - w;
            H.hi[a] = hi + w;
        }
        int32_t node = 0, res = -2;
        if (b.n_faces > 0) {
            while (true) {
                const QNode q = load_q(b, node);
                const float lx[4] = {q.lox.x, q.lox.y, q.lox.z, q.lox.w}, ly[4] = {q.loy.x, q.loy.y, q.loy.z, q.loy.w};
                const float lz[4] = {q.loz.x, q.loz.y, q.loz.z, q.loz.w}, hx[4] = {q.hix.x, q.hix.y, q.hix.z, q.hix.w};
                const float hy[4] = {q.hiy.x, q.hiy.y, q.hiy.z, q.hiy.w}, hz[4] = {q.hiz.x, q.hiz.y, q.hiz.z, q.hiz.w};
                int cnt = 0, only = -1;
                for (int k = 0; k < 4; ++k)
                    if (!hull_apart(H, lx[k], ly[k], lz[k], hx[k], hy[k], hz[k])) { ++cnt; only = k; }
                if (cnt == 0) { res = -2; break; }
                if (cnt == 1 && qref(q, only) >= 0) { node = qref(q, only); continue; }
                res = node;
                break;
            }
        }
        out[e] = res;
    }
}

}  // namespace bvh
