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
constexpr int kStack = 64;   // the host builder caps the tree depth below this

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

}  // namespace bvh
