// bvh_build.cpp - host BVH construction and refit (native runtime side of
// K2/K3/K11).
//
// The reference builds a longest-axis median-split BVH in Python
// (surface.py:320-369) and rebuilds it every simulation frame
// (scene.py:475-479). Hit results never depend on the tree (nearest t, ties
// to the smaller face id), so this builder is free to optimise for GPU
// traversal: 16-bin SAH over centroids, leaves of at most 4 faces, children
// stored as adjacent pairs, triangles re-laid out in leaf order, depth capped
// so the device short stack (bvh.cuh kStack) can never overflow.
#include "bvh_build.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

namespace hrt {

namespace {

constexpr int kBins = 16;
#ifndef HRT_BVH_LEAF
#define HRT_BVH_LEAF 1
#endif
constexpr int kLeaf = HRT_BVH_LEAF;   // max triangles per leaf (<= 7: 3-bit count in WNode refs)
constexpr int kSahDepth = 32;   // median splits below this: depth <= 32 + log2(n/4) < kStack

struct Box {
    double lo[3] = {std::numeric_limits<double>::infinity(), std::numeric_limits<double>::infinity(),
                    std::numeric_limits<double>::infinity()};
    double hi[3] = {-std::numeric_limits<double>::infinity(), -std::numeric_limits<double>::infinity(),
                    -std::numeric_limits<double>::infinity()};
    void grow(const Box& b) {
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], b.lo[a]); hi[a] = std::max(hi[a], b.hi[a]); }
    }
    void grow(const double* p) {
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], p[a]); hi[a] = std::max(hi[a], p[a]); }
    }
    double area() const {
        if (lo[0] > hi[0]) return 0.0;
        const double x = hi[0] - lo[0], y = hi[1] - lo[1], z = hi[2] - lo[2];
        return 2.0 * (x * y + y * z + z * x);
    }
};

// Face box padded for Moller-Trumbore's barycentric tolerance (hits may lie
// up to 1e-7 of an edge outside the face) and for rounding of v0 + e.
Box face_box(const double* v0, const double* e1, const double* e2) {
    Box b;
    double v1[3], v2[3];
    for (int a = 0; a < 3; ++a) { v1[a] = v0[a] + e1[a]; v2[a] = v0[a] + e2[a]; }
    b.grow(v0); b.grow(v1); b.grow(v2);
    double ext = 0.0, mag = 1.0;
    for (int a = 0; a < 3; ++a) {
        ext = std::max(ext, b.hi[a] - b.lo[a]);
        mag = std::max(mag, std::max(std::fabs(b.lo[a]), std::fabs(b.hi[a])));
    }
    const double pad = 1e-6 * ext + 1e-12 * mag;
    for (int a = 0; a < 3; ++a) { b.lo[a] -= pad; b.hi[a] += pad; }
    return b;
}

struct Builder {
    const double *v0, *e1, *e2;
    std::vector<Box> boxes;
    std::vector<double> cent;     // 3 per face
    std::vector<int32_t> idx;
    std::vector<BvhNodeHost> nodes;

    void set_leaf(int32_t node, int32_t begin, int32_t end) {
        nodes[node].first = begin;
        nodes[node].count = end - begin;
    }

    // Returns split position in idx[begin, end) or -1 for a leaf.
    int32_t split(int32_t begin, int32_t end, const Box& cb) {
        const int32_t n = end - begin;
        int axis = 0;
        double ext[3];
        for (int a = 0; a < 3; ++a) ext[a] = cb.hi[a] - cb.lo[a];
        if (ext[1] > ext[axis]) axis = 1;
        if (ext[2] > ext[axis]) axis = 2;
        if (!(ext[axis] > 0.0)) {       // coincident centroids: split in the middle
            return begin + n / 2;
        }
        Box bin_box[kBins];
        int32_t bin_cnt[kBins] = {0};
        const double k = kBins * (1.0 - 1e-9) / ext[axis];
        auto bin_of = [&](int32_t f) {
            int b = (int)((cent[3 * f + axis] - cb.lo[axis]) * k);
            return std::min(std::max(b, 0), kBins - 1);
        };
        for (int32_t i = begin; i < end; ++i) {
            const int b = bin_of(idx[i]);
            bin_cnt[b]++;
            bin_box[b].grow(boxes[idx[i]]);
        }
        double right_area[kBins];
        int32_t right_cnt[kBins];
        Box acc;
        int32_t cnt = 0;
        for (int b = kBins - 1; b > 0; --b) {
            acc.grow(bin_box[b]);
            cnt += bin_cnt[b];
            right_area[b] = acc.area();
            right_cnt[b] = cnt;
        }
        Box lacc;
        int32_t lcnt = 0;
        double best = std::numeric_limits<double>::infinity();
        int best_b = -1;
        for (int b = 1; b < kBins; ++b) {
            lacc.grow(bin_box[b - 1]);
            lcnt += bin_cnt[b - 1];
            if (lcnt == 0 || right_cnt[b] == 0) continue;
            const double cost = lacc.area() * lcnt + right_area[b] * right_cnt[b];
            if (cost < best) { best = cost; best_b = b; }
        }
        if (best_b < 0) return begin + n / 2;
        auto mid = std::partition(idx.begin() + begin, idx.begin() + end,
                                  [&](int32_t f) { return bin_of(f) < best_b; });
        int32_t m = (int32_t)(mid - idx.begin());
        if (m == begin || m == end) m = begin + n / 2;
        return m;
    }

    void build(int32_t n) {
        boxes.resize(n);
        cent.resize(3 * (size_t)n);
        idx.resize(n);
        for (int32_t f = 0; f < n; ++f) {
            boxes[f] = face_box(v0 + 3 * (size_t)f, e1 + 3 * (size_t)f, e2 + 3 * (size_t)f);
            for (int a = 0; a < 3; ++a) cent[3 * f + a] = 0.5 * (boxes[f].lo[a] + boxes[f].hi[a]);
            idx[f] = f;
        }
        nodes.reserve(2 * (size_t)n / kLeaf + 2);
        nodes.push_back({});
        struct Item { int32_t node, begin, end, depth; };
        std::vector<Item> stack{{0, 0, n, 0}};
        while (!stack.empty()) {
            const Item it = stack.back();
            stack.pop_back();
            Box nb, cb;
            for (int32_t i = it.begin; i < it.end; ++i) {
                nb.grow(boxes[idx[i]]);
                cb.grow(&cent[3 * (size_t)idx[i]]);
            }
            for (int a = 0; a < 3; ++a) { nodes[it.node].lo[a] = nb.lo[a]; nodes[it.node].hi[a] = nb.hi[a]; }
            const int32_t cnt = it.end - it.begin;
            if (cnt <= kLeaf) { set_leaf(it.node, it.begin, it.end); continue; }
            int32_t m;
            if (it.depth >= kSahDepth) {
                // force balanced median splits near the depth cap
                int axis = 0;
                for (int a = 1; a < 3; ++a)
                    if (cb.hi[a] - cb.lo[a] > cb.hi[axis] - cb.lo[axis]) axis = a;
                m = it.begin + cnt / 2;
                std::nth_element(idx.begin() + it.begin, idx.begin() + m, idx.begin() + it.end,
                                 [&](int32_t x, int32_t y) { return cent[3 * x + axis] < cent[3 * y + axis]; });
            } else {
                m = split(it.begin, it.end, cb);
            }
            const int32_t left = (int32_t)nodes.size();
            nodes.push_back({});
            nodes.push_back({});
            nodes[it.node].first = left;
            nodes[it.node].count = 0;
            stack.push_back({left + 1, m, it.end, it.depth + 1});
            stack.push_back({left, it.begin, m, it.depth + 1});
        }
    }
};

}  // namespace

BvhHost build_bvh(int64_t n_faces, const double* v0, const double* e1, const double* e2) {
    BvhHost out;
    out.n_faces = (int32_t)n_faces;
    if (n_faces == 0) return out;
    Builder b{v0, e1, e2};
    b.build((int32_t)n_faces);
    out.nodes = std::move(b.nodes);
    out.tri.resize(9 * (size_t)n_faces);
    out.tri_id.resize(n_faces);
    for (int32_t i = 0; i < (int32_t)n_faces; ++i) {
        const int32_t f = b.idx[i];
        std::memcpy(&out.tri[9 * (size_t)i], v0 + 3 * (size_t)f, 3 * sizeof(double));
        std::memcpy(&out.tri[9 * (size_t)i + 3], e1 + 3 * (size_t)f, 3 * sizeof(double));
        std::memcpy(&out.tri[9 * (size_t)i + 6], e2 + 3 * (size_t)f, 3 * sizeof(double));
        out.tri_id[i] = f;
    }
    out.parent.assign(out.nodes.size(), -1);
    for (size_t ni = 0; ni < out.nodes.size(); ++ni) {
        const BvhNodeHost& nd = out.nodes[ni];
        if (nd.count > 0) {
            out.leaves.push_back((int32_t)ni);
        } else {
            out.parent[nd.first] = (int32_t)ni;
            out.parent[nd.first + 1] = (int32_t)ni;
        }
    }
    return out;
}

BvhHost build_forest(int64_t n_faces, const double* v0, const double* e1, const double* e2,
                     const std::vector<int32_t>& group_begin) {
    BvhHost out;
    out.n_faces = (int32_t)n_faces;
    for (size_t g = 0; g + 1 < group_begin.size(); ++g) {
        const int32_t f0 = group_begin[g], nf = group_begin[g + 1] - f0;
        if (nf <= 0) continue;
        BvhHost t = build_bvh(nf, v0 + 3 * (size_t)f0, e1 + 3 * (size_t)f0, e2 + 3 * (size_t)f0);
        const int32_t noff = (int32_t)out.nodes.size(), toff = (int32_t)out.tri_id.size();
        out.roots.push_back(noff);
        for (size_t i = 0; i < t.nodes.size(); ++i) {
            BvhNodeHost nd = t.nodes[i];
            nd.first += nd.count > 0 ? toff : noff;
            out.nodes.push_back(nd);
            out.parent.push_back(t.parent[i] < 0 ? -1 : t.parent[i] + noff);
        }
        for (int32_t l : t.leaves) out.leaves.push_back(l + noff);
        out.tri.insert(out.tri.end(), t.tri.begin(), t.tri.end());
        for (int32_t id : t.tri_id) out.tri_id.push_back(id + f0);
    }
    return out;
}

}  // namespace hrt
