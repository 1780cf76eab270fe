// hrt.cu - C ABI implementation (include/hrt.h): scene upload, BVH build,
// weight packing, occupancy build, and the per-frame wavefront schedule.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hrt.h"
#include "bvh_build.h"
#include "kernels.cuh"
#include "probe.cuh"
#include <nvtx3/nvToolsExt.h>
#include "finalize.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(HRT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

#ifndef HRT_MAX_PATHS_LOG2
#define HRT_MAX_PATHS_LOG2 23
#endif
constexpr int64_t kMaxPaths = int64_t(1) << HRT_MAX_PATHS_LOG2;   // paths per wavefront chunk
// ... except for F = 4 fields (cfg4): 2^23-path chunks measured 1357 vs 1309 ms per
// 960x540x64 frame there, while cfg3 gains from them (193.8 vs 195.3 ms: two chunks of
// tail rounds and k_paths launches instead of four)
constexpr int64_t kMaxPathsF4 = std::min<int64_t>(kMaxPaths, int64_t(1) << 22);
constexpr int kThreads = 256;
#ifndef HRT_STEP_THREADS
#define HRT_STEP_THREADS 128
#endif
constexpr int kStepThreads = HRT_STEP_THREADS;     // k_step block size
constexpr int kTimedLaunches = 1024;
constexpr int kIoChunks = 4;                       // pieces of the e2e frame read-back
#ifndef HRT_SHADOW_QUEUE
#define HRT_SHADOW_QUEUE 1
#endif
constexpr bool kShadowQueue = HRT_SHADOW_QUEUE;   // shadow rays: set-up pass + persistent tracer
// Batch rows per march round: 2^27 lets a full 2^22-path chunk take up to 32 samples per
// path in its first rounds (2^26 capped them at 16): cfg3 frame 196.5 -> 195.8 ms, cfg4
// 960x540x64 1314 -> 1309 ms; a 2^23-path chunk (F = 2) takes up to 16 in its first rounds
#ifndef HRT_BATCH_CAP_LOG2
#define HRT_BATCH_CAP_LOG2 27
#endif
constexpr int64_t kBatchCap = int64_t(1) << HRT_BATCH_CAP_LOG2;   // samples per march round
#ifndef HRT_TEX_LEVELS
#define HRT_TEX_LEVELS 8
#endif
constexpr int kTexLevels = HRT_TEX_LEVELS;        // finest levels gathered via TEX
#ifndef HRT_TEAM_TEX_LEVELS
#define HRT_TEAM_TEX_LEVELS 12
#endif
// ... in the encode-team (coherent) rounds of an F = 2 field: 10-16 TEX levels there
// measured equal and 2 ms faster per cfg3 frame than 8 (F = 4: 8 stays best)
constexpr int kTeamTexLevels = HRT_TEAM_TEX_LEVELS;
#ifndef HRT_TEAM_ROUNDS
#define HRT_TEAM_ROUNDS 3
#endif
constexpr int kTeamRounds = HRT_TEAM_ROUNDS;       // march rounds run with encode teams (fws T >= 2)
#ifndef HRT_TEAMS_F2
#define HRT_TEAMS_F2 2
#endif
constexpr int kTeamsF2 = HRT_TEAMS_F2;            // encode teams in the E = 32, F = 2 team rounds
#ifndef HRT_TEAM_ROUNDS_F4
#define HRT_TEAM_ROUNDS_F4 5
#endif
constexpr int kTeamRoundsF4 = HRT_TEAM_ROUNDS_F4;  // ... for F = 4 fields (cfg4 960x540x64: 3 / 5 / 8 rounds
                                                   // 640 / 631 / 640 ms field)
// encode teams also for F = 4 fields (cfg4 960x540x64: field 670 -> 641 ms, despite
// 76 B of spills in k_field_ws<64, 4, 2>)
#ifndef HRT_TEAMS_F4
#define HRT_TEAMS_F4 1
#endif
constexpr bool kTeamsF4 = HRT_TEAMS_F4;
#ifndef HRT_PATHS_BY_BOUNCE
#define HRT_PATHS_BY_BOUNCE 1
#endif
constexpr bool kPathsByBounce = HRT_PATHS_BY_BOUNCE;   // k_paths_bounce per bounce (compacted) vs k_paths
#ifndef HRT_MIXED_MARCH
#define HRT_MIXED_MARCH 1
#endif
constexpr bool kMixedMarch = HRT_MIXED_MARCH;     // continuous wavefront march (kern::advance)
#ifndef HRT_COOP_PATHS
#define HRT_COOP_PATHS 200000
#endif
constexpr int64_t kCoopPaths = HRT_COOP_PATHS;     // k_paths_coop (4 lanes per path) below this
#ifndef HRT_TILED_FRAME
#define HRT_TILED_FRAME 1
#endif
constexpr bool kTiledFrame = HRT_TILED_FRAME;      // full frames walk 16x16 pixel tiles

}  // namespace

struct RefitState {              // device side of a BVH's GPU refit
    int2* wsrc = nullptr;        // float64 node behind each WNode child slot
    int32_t n_w = 0;
    int32_t w_begin = 0;         // forest: WNodes [0, w_begin) are the top level over the roots
    std::vector<int32_t> roots;  // forest: root node of every group's tree
    std::vector<int32_t> root_ref;   // and its WNode reference
    int32_t* d_roots = nullptr;
    double* d_rootbox = nullptr; // gathered root boxes (6 doubles each)
    int4* qsrc = nullptr;        // float64 node behind each QNode child slot
    int32_t n_q = 0, q_begin = 0;    // forest: QNodes [0, q_begin) hold the top level
    std::vector<int32_t> qmap;   // WNode index -> QNode index of every tree root (forest)
    int32_t* parent = nullptr;
    int32_t* leaves = nullptr;
    int32_t* visits = nullptr;
    double* src = nullptr;         // staging: v0 | e1 | e2 in global face order
    int32_t n_leaves = 0;
};

struct hrt_handle {
    DevScene sc{};
    RefitState rf, rfb;
    std::vector<void*> allocs;
    std::vector<cudaTextureObject_t> texs;   // BVH node textures (upload_bvh)
    hrt::BvhHost bvh, blk;
    BvhNode* d_nodes = nullptr;
    double* d_tri = nullptr;
    BvhNode* d_bnodes = nullptr;
    double* d_btri = nullptr;
    double* d_normal = nullptr;
    int E = 0, F = 0;
    int sm_count = 148;
    // path-state arena
    int64_t cap = 0;
    void* arena = nullptr;
    PathState ps{};
    int32_t* trace = nullptr;
    int64_t trace_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t mev[2 * 1024] = {};
    int64_t* round_rows = nullptr;  // device: batch rows of each device-driven march round (k_round_begin)
    int32_t n_round_rows = 0;       // rounds logged by the last render call
    kern::MarchState ms{};
    int64_t batch_cap = 0;
    int32_t* pinned = nullptr;
    int64_t rounds = 0;
    int64_t batch_rows = 0;
    int64_t io_cap = 0;
    int32_t *io_pix = nullptr, *io_pix_host = nullptr;
    double *io_out = nullptr, *io_out_host = nullptr;
    cudaStream_t io_stream = nullptr;
    cudaEvent_t io_ev[8] = {};
    int n_timed = 0;
    int64_t launches = 0;
    uint32_t* occ_dev = nullptr;
    int64_t occ_words = 0;
    unsigned long long tex = 0;
    double* rigid_xf = nullptr;     // hrt_refit_rigid: device copy of the per-mesh transforms
    int32_t rigid_xf_cap = 0;
    bool blk_stale = false;         // blocker forest behind the last hrt_refit_rigid (no emitters)
    double* rigid_base = nullptr;   // hrt_set_rigid_base: object-space corners, global face order
    std::vector<int32_t> mesh_of_host;
    int32_t n_meshes = 0;           // max(mesh_of) + 1
    int32_t* blk_map = nullptr;     // blocker face -> global face
    int64_t tab_entries = 0;
    int shadow_blocks = 0;
    // hrt_set_profile: event pair per launch, folded into stage_ms
    bool prof = false;
    bool continuous = kMixedMarch;   // hrt_set_march
    // shadow entry table (bvh::k_shadow_entry): rebuilt when the blocker
    // tree or the field placement changed (geo_ver) since it was made
    int32_t* shent = nullptr;
    int64_t shent_n = 0;
    int64_t geo_ver = 0, shent_ver = -1;
    bool shent_on = true;            // HRT_SHADOW_ENTRY=0 at create: off
    void* geo_arena = nullptr;       // kern::PathGeo storage (ensure_geo)
    int64_t geo_n = 0;
    std::vector<cudaEvent_t> pev;
    std::vector<int> pstage;
    int pn = 0;
    double stage_ms[8] = {};

    template <class T>
    int upload(const T* src, size_t n, T** dst) {
        *dst = nullptr;
        if (n == 0 || src == nullptr) return HRT_OK;
        void* p = nullptr;
        CK(cudaMalloc(&p, n * sizeof(T)));
        allocs.push_back(p);
        CK(cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
        *dst = static_cast<T*>(p);
        return HRT_OK;
    }
    int alloc(size_t bytes, void** dst) {
        CK(cudaMalloc(dst, bytes));
        allocs.push_back(*dst);
        return HRT_OK;
    }
    ~hrt_handle() {
        for (void* p : allocs) cudaFree(p);
        if (arena) cudaFree(arena);
        if (geo_arena) cudaFree(geo_arena);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (cudaEvent_t e : mev) if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : pev) cudaEventDestroy(e);
        if (pinned) cudaFreeHost(pinned);
        if (rigid_xf) cudaFree(rigid_xf);
        if (shent) cudaFree(shent);
        if (io_pix) cudaFree(io_pix);
        if (io_out) cudaFree(io_out);
        if (io_pix_host) cudaFreeHost(io_pix_host);
        if (io_out_host) cudaFreeHost(io_out_host);
        if (io_stream) cudaStreamDestroy(io_stream);
        for (cudaEvent_t e : io_ev) if (e) cudaEventDestroy(e);
        if (tex) cudaDestroyTextureObject(tex);
        for (cudaTextureObject_t t : texs) cudaDestroyTextureObject(t);
    }
};

namespace {

int setup_refit(hrt_handle* h, const hrt::BvhHost& b, RefitState& r) {
    if (b.n_faces == 0) return HRT_OK;
    int rc;
    if ((rc = h->upload(b.parent.data(), b.parent.size(), &r.parent))) return rc;
    if ((rc = h->upload(b.leaves.data(), b.leaves.size(), &r.leaves))) return rc;
    if ((rc = h->alloc(b.nodes.size() * 4, reinterpret_cast<void**>(&r.visits)))) return rc;
    if ((rc = h->alloc((size_t)b.n_faces * 9 * 8, reinterpret_cast<void**>(&r.src)))) return rc;
    r.n_leaves = (int32_t)b.leaves.size();
    return HRT_OK;
}

// K11: upload the new world-space faces, permute them into leaf order and
// refit the boxes bottom-up on the device.
int refit_from_src(hrt_handle* h, const hrt::BvhHost& b, RefitState& r, DevBvh& dev);
void build_tlas(const std::vector<hrt::BvhNodeHost>& box, const std::vector<int32_t>& ref, WNode* w);
void collapse_top(const std::vector<WNode>& top, RefitState& r, std::vector<QNode>& Q);

int refit_gpu(hrt_handle* h, const hrt::BvhHost& b, RefitState& r, DevBvh& dev, const double* v0,
              const double* e1, const double* e2) {
    const size_t n3 = 3 * (size_t)b.n_faces;
    CK(cudaMemcpy(r.src, v0, n3 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(r.src + n3, e1, n3 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(r.src + 2 * n3, e2, n3 * 8, cudaMemcpyHostToDevice));
    return refit_from_src(h, b, r, dev);
}

// Refit from faces already in r.src (v0 | e1 | e2, global face order).
int refit_from_src(hrt_handle* h, const hrt::BvhHost& b, RefitState& r, DevBvh& dev) {
    ++h->geo_ver;
    const size_t n3 = 3 * (size_t)b.n_faces;
    CK(cudaMemset(r.visits, 0, b.nodes.size() * 4));
    const unsigned g1 = (unsigned)std::min<int64_t>((b.n_faces + 255) / 256, 148 * 16);
    bvh::k_permute_tris<<<g1, 256>>>(r.src, r.src + n3, r.src + 2 * n3, dev.tri_id, b.n_faces,
                                     const_cast<double*>(dev.tri));
    CK(cudaGetLastError());
    const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((r.n_leaves + 255) / 256, 148 * 16));
    bvh::k_refit<<<g2, 256>>>(const_cast<BvhNode*>(dev.nodes), r.parent, r.leaves, r.n_leaves, dev.tri,
                              r.visits);
    CK(cudaGetLastError());
    const unsigned g3 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((r.n_w + 255) / 256, 148 * 16));
    bvh::k_wsync<<<g3, 256>>>(const_cast<WNode*>(dev.wnodes), r.wsrc, dev.nodes, r.w_begin, r.n_w);
    CK(cudaGetLastError());
    const unsigned g4 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((r.n_q + 255) / 256, 148 * 16));
    bvh::k_qsync<<<g4, 256>>>(const_cast<QNode*>(dev.qnodes), r.qsrc, dev.nodes, r.q_begin, r.n_q);
    CK(cudaGetLastError());
    if (!r.roots.empty()) {          // forest: new root boxes -> rebuild the top level
        const int32_t G = (int32_t)r.roots.size();
        bvh::k_root_boxes<<<(G + 255) / 256, 256>>>(dev.nodes, r.d_roots, G, r.d_rootbox);
        CK(cudaGetLastError());
        std::vector<double> rb(6 * (size_t)G);
        CK(cudaMemcpy(rb.data(), r.d_rootbox, rb.size() * 8, cudaMemcpyDeviceToHost));
        std::vector<hrt::BvhNodeHost> boxes(G);
        for (int32_t g = 0; g < G; ++g)
            for (int a = 0; a < 3; ++a) {
                boxes[g].lo[a] = rb[6 * g + a];
                boxes[g].hi[a] = rb[6 * g + 3 + a];
            }
        std::vector<WNode> top(G - 1);
        build_tlas(boxes, r.root_ref, top.data());
        CK(cudaMemcpy(const_cast<WNode*>(dev.wnodes), top.data(), top.size() * sizeof(WNode),
                      cudaMemcpyHostToDevice));
        std::vector<QNode> qtop;
        collapse_top(top, r, qtop);
        CK(cudaMemcpy(const_cast<QNode*>(dev.qnodes), qtop.data(), qtop.size() * sizeof(QNode),
                      cudaMemcpyHostToDevice));
    }
    return HRT_OK;
}

// float64 -> float32 rounded toward -inf / +inf (device: __double2float_rd/ru)
float f_rd(double x) {
    float f = (float)x;
    if ((double)f > x) f = std::nextafter(f, -INFINITY);
    return f;
}
float f_ru(double x) {
    float f = (float)x;
    if ((double)f < x) f = std::nextafter(f, INFINITY);
    return f;
}

// Child box of a WNode: the float64 node box padded by 1e-5 * max(1, |coord|)
// and rounded outward (same rule as bvh.cuh wbox_dev, used after refits).
void wbox(const hrt::BvhNodeHost& n, float lo[3], float hi[3]) {
    double mag = 1.0;
    for (int a = 0; a < 3; ++a) mag = std::max(mag, std::max(std::fabs(n.lo[a]), std::fabs(n.hi[a])));
    const double pad = 1e-5 * mag;
    for (int a = 0; a < 3; ++a) {
        lo[a] = f_rd(n.lo[a] - pad);
        hi[a] = f_ru(n.hi[a] + pad);
    }
}

void wset(WNode& x, const hrt::BvhNodeHost* n0, const hrt::BvhNodeHost* n1, int32_t r0, int32_t r1) {
    float l0[3], h0[3], l1[3], h1[3];
    for (int a = 0; a < 3; ++a) l0[a] = h0[a] = l1[a] = h1[a] = 1e30f;
    if (n0) wbox(*n0, l0, h0);
    if (n1) wbox(*n1, l1, h1);
    x.a = make_float4(l0[0], l0[1], l0[2], h0[0]);
    x.b = make_float4(h0[1], h0[2], l1[0], l1[1]);
    x.c = make_float4(l1[2], h1[0], h1[1], h1[2]);
    x.r = make_int4(r0, r1, 0, 0);
}

// Top level of a forest over its G root boxes: G-1 WNodes written to w[0..),
// root at 0, median splits on the widest centroid axis (rebuilt per frame).
void build_tlas(const std::vector<hrt::BvhNodeHost>& box, const std::vector<int32_t>& ref, WNode* w) {
    std::vector<int32_t> it(box.size());
    for (size_t i = 0; i < it.size(); ++i) it[i] = (int32_t)i;
    int32_t next = 0;
    std::function<std::pair<int32_t, hrt::BvhNodeHost>(int32_t, int32_t)> rec =
        [&](int32_t b, int32_t e) -> std::pair<int32_t, hrt::BvhNodeHost> {
        if (e - b == 1) return {ref[it[b]], box[it[b]]};
        const int32_t t = next++;
        double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int32_t i = b; i < e; ++i)
            for (int a = 0; a < 3; ++a) {
                const double c = 0.5 * (box[it[i]].lo[a] + box[it[i]].hi[a]);
                clo[a] = std::min(clo[a], c);
                chi[a] = std::max(chi[a], c);
            }
        int ax = 0;
        for (int a = 1; a < 3; ++a)
            if (chi[a] - clo[a] > chi[ax] - clo[ax]) ax = a;
        const int32_t m = b + (e - b) / 2;
        std::nth_element(it.begin() + b, it.begin() + m, it.begin() + e, [&](int32_t x, int32_t y) {
            return box[x].lo[ax] + box[x].hi[ax] < box[y].lo[ax] + box[y].hi[ax];
        });
        auto L = rec(b, m), R = rec(m, e);
        wset(w[t], &L.second, &R.second, L.first, R.first);
        hrt::BvhNodeHost u;
        for (int a = 0; a < 3; ++a) {
            u.lo[a] = std::min(L.second.lo[a], R.second.lo[a]);
            u.hi[a] = std::max(L.second.hi[a], R.second.hi[a]);
        }
        return {t, u};
    };
    rec(0, (int32_t)box.size());
}

// ---- 4-wide traversal tree: the binary WNode tree collapsed (each QNode
// takes a WNode's two children and expands inner ones, largest area first,
// until it has 4 slots). Boxes are copied, so culling stays conservative.
struct QSlot {
    float lo[3], hi[3];
    int32_t ref, src;
};

QSlot wslot(const WNode& w, const int2& s, int k) {
    QSlot q;
    if (k == 0) {
        q.lo[0] = w.a.x; q.lo[1] = w.a.y; q.lo[2] = w.a.z;
        q.hi[0] = w.a.w; q.hi[1] = w.b.x; q.hi[2] = w.b.y;
        q.ref = w.r.x; q.src = s.x;
    } else {
        q.lo[0] = w.b.z; q.lo[1] = w.b.w; q.lo[2] = w.c.x;
        q.hi[0] = w.c.y; q.hi[1] = w.c.z; q.hi[2] = w.c.w;
        q.ref = w.r.y; q.src = s.y;
    }
    return q;
}

double qarea(const QSlot& q) {
    double e[3];
    for (int a = 0; a < 3; ++a) e[a] = std::max(0.0, (double)q.hi[a] - (double)q.lo[a]);
    return e[0] * e[1] + e[1] * e[2] + e[2] * e[0];
}

// Collapse WNode w into QNode index `at` (already reserved); children that
// `expand` accepts are collapsed recursively into indices taken from *next,
// other inner refs are translated with `map_inner`.
void qcollapse(const WNode* W, const int2* S, int32_t w, int32_t at, std::vector<QNode>& Q,
               std::vector<int4>& QS, int32_t* next, const std::function<bool(int32_t)>& expand,
               const std::function<int32_t(int32_t)>& map_inner) {
    std::vector<QSlot> sl = {wslot(W[w], S[w], 0), wslot(W[w], S[w], 1)};
    while (sl.size() < 4) {
        int best = -1;
        double ba = -1.0;
        for (size_t k = 0; k < sl.size(); ++k)
            if (sl[k].ref >= 0 && expand(sl[k].ref) && qarea(sl[k]) > ba) { ba = qarea(sl[k]); best = (int)k; }
        if (best < 0) break;
        const int32_t c = sl[best].ref;
        sl[best] = wslot(W[c], S[c], 0);
        sl.push_back(wslot(W[c], S[c], 1));
    }
    QNode q;
    float* f = reinterpret_cast<float*>(&q);
    int32_t refs[4] = {-1, -1, -1, -1}, srcs[4] = {-1, -1, -1, -1};
    for (int k = 0; k < 4; ++k)
        for (int a = 0; a < 3; ++a) { f[4 * a + k] = 1e30f; f[12 + 4 * a + k] = 1e30f; }
    std::vector<std::pair<int32_t, int32_t>> todo;       // (wnode, qnode) to collapse after this one
    for (size_t k = 0; k < sl.size(); ++k) {
        for (int a = 0; a < 3; ++a) { f[4 * a + k] = sl[k].lo[a]; f[12 + 4 * a + k] = sl[k].hi[a]; }
        srcs[k] = sl[k].src;
        if (sl[k].ref < 0) {
            refs[k] = sl[k].ref;
        } else if (expand(sl[k].ref)) {
            refs[k] = (*next)++;
            todo.push_back({sl[k].ref, refs[k]});
        } else {
            refs[k] = map_inner(sl[k].ref);
        }
    }
    q.ref = make_int4(refs[0], refs[1], refs[2], refs[3]);
    q.pad = make_int4(0, 0, 0, 0);
    if ((int32_t)Q.size() <= at) { Q.resize(at + 1); QS.resize(at + 1); }
    Q[at] = q;
    QS[at] = make_int4(srcs[0], srcs[1], srcs[2], srcs[3]);
    for (auto& t : todo) qcollapse(W, S, t.first, t.second, Q, QS, next, expand, map_inner);
}

// 4-wide tree of a built WNode array (single tree or forest), r.qmap / q_begin set.
void build_qnodes(const std::vector<WNode>& W, const std::vector<int2>& S, RefitState& r,
                  std::vector<QNode>& Q, std::vector<int4>& QS) {
    Q.clear();
    QS.clear();
    r.qmap.clear();
    const int32_t T = r.w_begin;
    if (r.roots.empty() || T == 0) {                   // one tree
        int32_t next = 1;
        qcollapse(W.data(), S.data(), 0, 0, Q, QS, &next, [](int32_t) { return true; },
                  [](int32_t c) { return c; });
        r.q_begin = 0;
        return;
    }
    // forest: trees first (from index T), then the top level into [0, T)
    r.qmap.assign(W.size(), -1);
    int32_t next = T;
    Q.resize(T);
    QS.assign(T, make_int4(-1, -1, -1, -1));
    for (int32_t rf : r.root_ref) {
        if (rf < 0) continue;                         // tree of one leaf: stays a leaf ref
        const int32_t at = next++;
        r.qmap[rf] = at;
        qcollapse(W.data(), S.data(), rf, at, Q, QS, &next, [T](int32_t c) { return c >= T; },
                  [](int32_t c) { return c; });
    }
    r.q_begin = T;
    int32_t top = 1;
    std::vector<int32_t>& qm = r.qmap;
    qcollapse(W.data(), S.data(), 0, 0, Q, QS, &top, [T](int32_t c) { return c < T; },
              [&qm](int32_t c) { return qm[c]; });
    for (int32_t i = 0; i < T; ++i) QS[i] = make_int4(-1, -1, -1, -1);   // top level: host-rebuilt
}

// Per-frame top level of a forest in QNodes [0, q_begin): collapse the
// rebuilt binary top level, tree roots mapped through qmap.
void collapse_top(const std::vector<WNode>& top, RefitState& r, std::vector<QNode>& Q) {
    const int32_t T = r.w_begin;
    std::vector<int2> S(T, make_int2(-1, -1));
    std::vector<int4> QS;
    Q.clear();
    int32_t next = 1;
    std::vector<int32_t>& qm = r.qmap;
    qcollapse(top.data(), S.data(), 0, 0, Q, QS, &next, [T](int32_t c) { return c < T; },
              [&qm](int32_t c) { return qm[c]; });
}

// float32-culling tree over the same leaves: one WNode per inner float64
// node (a root leaf gets a WNode with an empty second child); src records
// the float64 node behind each child slot for k_wsync after refits. A
// forest (b.roots, >= 2 trees) gets a top level over the roots in
// WNodes [0, G-1) (r.w_begin), its trees' WNodes after it.
void build_wnodes(const hrt::BvhHost& b, std::vector<WNode>& w, std::vector<int2>& src, RefitState& r) {
    const auto& nd = b.nodes;
    const bool forest = b.roots.size() >= 2;
    const int32_t T = forest ? (int32_t)b.roots.size() - 1 : 0;
    std::vector<int32_t> widx(nd.size(), -1);
    int32_t nw = T;
    for (size_t i = 0; i < nd.size(); ++i)
        if (nd[i].count == 0) widx[i] = nw++;
    auto ref = [&](int32_t c) -> int32_t {
        return nd[c].count > 0 ? ~((nd[c].first << 3) | nd[c].count) : widx[c];
    };
    r.w_begin = T;
    r.roots.clear();
    r.root_ref.clear();
    if (!forest && nd[0].count > 0) {           // whole mesh in one leaf
        w.assign(1, WNode{});
        src.assign(1, make_int2(0, -1));
        wset(w[0], &nd[0], nullptr, ref(0), -1);
        return;
    }
    w.assign(nw, WNode{});
    src.assign(nw, make_int2(-1, -1));
    for (size_t i = 0; i < nd.size(); ++i) {
        if (nd[i].count != 0) continue;
        const int32_t c = nd[i].first;
        wset(w[widx[i]], &nd[c], &nd[c + 1], ref(c), ref(c + 1));
        src[widx[i]] = make_int2(c, c + 1);
    }
    if (forest) {
        std::vector<hrt::BvhNodeHost> boxes;
        for (int32_t rt : b.roots) {
            r.roots.push_back(rt);
            r.root_ref.push_back(ref(rt));
            boxes.push_back(nd[rt]);
        }
        build_tlas(boxes, r.root_ref, w.data());
    }
}

int upload_bvh(hrt_handle* h, const hrt::BvhHost& b, DevBvh& out, RefitState& r) {
    ++h->geo_ver;
    out.n_faces = b.n_faces;
    out.nodes = nullptr; out.tri = nullptr; out.tri_id = nullptr; out.wnodes = nullptr; out.qnodes = nullptr;
    out.qtex = 0;
    r.wsrc = nullptr;
    r.n_w = 0;
    if (b.n_faces == 0) return HRT_OK;
    {
        std::vector<WNode> w;
        std::vector<int2> src;
        build_wnodes(b, w, src, r);
        WNode* dw;
        int rc;
        if ((rc = h->upload(w.data(), w.size(), &dw))) return rc;
        if ((rc = h->upload(src.data(), src.size(), &r.wsrc))) return rc;
        out.wnodes = dw;
        r.n_w = (int32_t)w.size();
        std::vector<QNode> q;
        std::vector<int4> qs;
        build_qnodes(w, src, r, q, qs);
        QNode* dq;
        if ((rc = h->upload(q.data(), q.size(), &dq))) return rc;
        if ((rc = h->upload(qs.data(), qs.size(), &r.qsrc))) return rc;
        out.qnodes = dq;
        r.n_q = (int32_t)q.size();
        {   // texture view of the nodes (bvh::load_q)
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeLinear;
            rd.res.linear.devPtr = dq;
            rd.res.linear.desc = cudaCreateChannelDesc<float4>();
            rd.res.linear.sizeInBytes = q.size() * sizeof(QNode);
            cudaTextureDesc td{};
            td.readMode = cudaReadModeElementType;
            td.filterMode = cudaFilterModePoint;
            cudaTextureObject_t to = 0;
            CK(cudaCreateTextureObject(&to, &rd, &td, nullptr));
            h->texs.push_back(to);
            out.qtex = to;
        }
        if (!r.roots.empty()) {
            if ((rc = h->upload(r.roots.data(), r.roots.size(), &r.d_roots))) return rc;
            if ((rc = h->alloc(r.roots.size() * 6 * 8, reinterpret_cast<void**>(&r.d_rootbox)))) return rc;
        }
    }
    static_assert(sizeof(BvhNode) == sizeof(hrt::BvhNodeHost), "node layout");
    BvhNode* nodes;
    double* tri;
    int32_t* ids;
    int rc;
    if ((rc = h->upload(reinterpret_cast<const BvhNode*>(b.nodes.data()), b.nodes.size(), &nodes))) return rc;
    if ((rc = h->upload(b.tri.data(), b.tri.size(), &tri))) return rc;
    if ((rc = h->upload(b.tri_id.data(), b.tri_id.size(), &ids))) return rc;
    out.nodes = nodes; out.tri = tri; out.tri_id = ids;

    return HRT_OK;
}

// fp16 weights [K_in][N_out] row-major -> UMMA B image (N_pad x K_pad,
// K-major core matrices), zero padded.
void pack_layer(const uint16_t* w, int k_in, int n_out, int K, int N, uint8_t* dst) {
    std::memset(dst, 0, (size_t)K * N * 2);
    for (int n = 0; n < n_out; ++n)
        for (int k = 0; k < k_in; ++k) {
            const size_t off = (size_t)(n >> 3) * (K * 16) + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
            std::memcpy(dst + off, &w[(size_t)k * n_out + n], 2);
        }
}

int setup_field(hrt_handle* h, const hrt_field_desc& fd) {
    DevField& f = h->sc.field;
    f.kind = fd.kind;
    f.identity = fd.identity;
    for (int a = 0; a < 3; ++a) { f.lo[a] = fd.bbox_lo[a]; f.hi[a] = fd.bbox_hi[a]; }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 4; ++c) f.inv[4 * r + c] = fd.field_from_world[4 * r + c];
    int rc;
    if (fd.kind == HRT_FIELD_DENSE) {
        DenseGrid& g = f.dense;
        const size_t n = (size_t)fd.res[0] * fd.res[1] * fd.res[2];
        if (n == 0 || !fd.sigma || !fd.radiance) return fail(HRT_EINVAL, "dense field needs sigma/radiance");
        for (int a = 0; a < 3; ++a) { g.res[a] = fd.res[a]; g.scale[a] = fd.scale[a]; }
        double *s, *r;
        if ((rc = h->upload(fd.sigma, n, &s))) return rc;
        if ((rc = h->upload(fd.radiance, 3 * n, &r))) return rc;
        g.sigma = s; g.rad = r;
        g.sigma_const = fd.sigma_const; g.rad_const = fd.rad_const;
        g.sigma0 = fd.sigma[0];
        for (int c = 0; c < 3; ++c) g.rad0[c] = fd.radiance[c];
    } else if (fd.kind == HRT_FIELD_NEURAL) {
        NeuralField& nf = f.nf;
        const int L = fd.n_levels, F = fd.n_features;
        if (L < 1 || L > kMaxLevels || (F != 2 && F != 4)) return fail(HRT_EINVAL, "bad hash-grid shape");
        const int E = L * F;
        if (E != 16 && E != 32 && E != 64) return fail(HRT_EINVAL, "L*F must be 16, 32 or 64");
        h->E = E; h->F = F;
        nf.n_levels = L; nf.n_features = F; nf.enc_dim = E; nf.act = fd.act;
        nf.tmask = (uint32_t)((1ull << fd.log2_table) - 1);
        for (int a = 0; a < 3; ++a) nf.lo32[a] = (float)fd.bbox_lo[a];
        // Device table: same entries, each level starting on an even entry
        // (16-byte aligned pairs for the x-pair gathers in encode_level), and
        // every hashed level on a multiple of T entries, so that its offset
        // folds into the hash with an OR (nerf::level_issue).
        const int64_t T = int64_t(1) << fd.log2_table;
        int64_t padded = 0;
        std::vector<int64_t> dev_off(L);
        for (int l = 0; l < L; ++l) {
            const int64_t end = l + 1 < L ? fd.level_offset[l + 1] : fd.n_entries;
            if (!fd.level_dense[l]) {
                if (end - fd.level_offset[l] > T) return fail(HRT_EINVAL, "hashed level larger than T");
                padded = (padded + T - 1) / T * T;
            }
            dev_off[l] = padded;
            padded += ((end - fd.level_offset[l]) + 1) & ~int64_t(1);
        }
        if (padded >= (int64_t(1) << 31)) return fail(HRT_EINVAL, "hash table too large");
        std::vector<float> tab((size_t)padded * F, 0.0f);
        for (int l = 0; l < L; ++l) {
            NeuralLevel& lv = nf.lv[l];
            for (int a = 0; a < 3; ++a) lv.scale[a] = fd.level_scale[3 * l + a];
            lv.n = fd.level_n[l];
            lv.r = (uint32_t)fd.level_n[l] + 1;
            lv.dense = fd.level_dense[l];
            lv.offset = dev_off[l];
            const int64_t end = l + 1 < L ? fd.level_offset[l + 1] : fd.n_entries;
            std::memcpy(&tab[(size_t)dev_off[l] * F], fd.table + (size_t)fd.level_offset[l] * F,
                        (size_t)(end - fd.level_offset[l]) * F * sizeof(float));
        }
        float* table;
        if ((rc = h->upload(tab.data(), tab.size(), &table))) return rc;
        h->tab_entries = padded;
        nf.table = table;
        {   // texture view of the table: the finest (incoherent) levels gather through the
            // TEX pipe of L1TEX, the rest through LSU, splitting the data-stage load
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeLinear;
            rd.res.linear.devPtr = table;
            rd.res.linear.desc = F == 2 ? cudaCreateChannelDesc<float2>() : cudaCreateChannelDesc<float4>();
            rd.res.linear.sizeInBytes = tab.size() * sizeof(float);
            cudaTextureDesc td{};
            td.readMode = cudaReadModeElementType;
            td.filterMode = cudaFilterModePoint;
            cudaTextureObject_t to = 0;
            CK(cudaCreateTextureObject(&to, &rd, &td, nullptr));
            h->tex = to;
            nf.tex = to;
            nf.tex_from = std::max(0, L - kTexLevels);
        }
        const nerf::WOff W = nerf::woff(E);
        std::vector<uint8_t> img(W.total);
        pack_layer(fd.w_density1, E, 64, E, 64, img.data() + W.d1);
        pack_layer(fd.w_density2, 64, 16, 64, 16, img.data() + W.d2);
        pack_layer(fd.w_color1, 32, 64, 32, 64, img.data() + W.c1);
        pack_layer(fd.w_color2, 64, 64, 64, 64, img.data() + W.c2);
        pack_layer(fd.w_color3, 64, 3, 64, 16, img.data() + W.c3);
        uint8_t* wp;
        if ((rc = h->upload(img.data(), img.size(), &wp))) return rc;
        nf.wpack = wp;
        const int G = fd.occ_res;
        nf.occ_res = G;
        for (int a = 0; a < 3; ++a) {
            nf.occ_scale[a] = fd.occ_scale[a];
            nf.occ_cell[a] = (fd.bbox_hi[a] - fd.bbox_lo[a]) / G;
        }
        h->occ_words = ((int64_t)G * G * G + 31) / 32;
        if (fd.occ_bits) {
            if ((rc = h->upload(fd.occ_bits, (size_t)h->occ_words, &h->occ_dev))) return rc;
        } else {
            if ((rc = h->alloc((size_t)h->occ_words * 4, reinterpret_cast<void**>(&h->occ_dev)))) return rc;
        }
        nf.occ = h->occ_dev;
    }
    return HRT_OK;
}

// ------------------------------------------------------------ field engine
unsigned grid_for(const hrt_handle* h, int64_t n) {
    const int64_t g = (n + kThreads - 1) / kThreads;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)h->sm_count * 16));
}

template <int E, int F, int T = 1>
int launch_ws(hrt_handle* h, const fws::SampleIn* in, fws::RowMap rm, int64_t n, const float4* dir32,
              float4* out, int density_only, const int32_t* round_ctr, cudaStream_t st) {
    constexpr uint32_t smem = fws::plan(E).total;
    CK(cudaFuncSetAttribute(fws::k_field_ws<E, F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t tiles = (n + fws::kRows - 1) / fws::kRows;
    const int grid = round_ctr ? h->sm_count
                               : (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)h->sm_count));
    NeuralField nf = h->sc.field.nf;
    if (T >= 2 && F == 2) nf.tex_from = std::max(0, nf.n_levels - kTeamTexLevels);
    fws::k_field_ws<E, F, T><<<grid, fws::kThreads, smem, st>>>(nf, in, rm, n, dir32, out,
                                                             density_only, round_ctr, h->ps.stats,
                                                             round_ctr ? h->round_rows : nullptr);
    CK(cudaGetLastError());
    return HRT_OK;
}

// Evaluate a batch of n logical rows (RowMap: where they live) with the
// field engine; bracketed by events so the dominant kernel's device time is
// measured live.
int field_ws(hrt_handle* h, const fws::SampleIn* in, fws::RowMap rm, int64_t n, const float4* dir32,
             float4* out, int density_only, cudaStream_t st, const int32_t* round_ctr = nullptr,
             bool teams = false) {
    if (n <= 0 && !round_ctr) return HRT_OK;
    const bool timed = h->n_timed < kTimedLaunches;
    if (timed) CK(cudaEventRecord(h->mev[2 * h->n_timed], st));
    int rc;
    switch (h->E * 8 + h->F) {
        case 16 * 8 + 2:
            rc = teams ? launch_ws<16, 2, 2>(h, in, rm, n, dir32, out, density_only, round_ctr, st)
                       : launch_ws<16, 2>(h, in, rm, n, dir32, out, density_only, round_ctr, st);
            break;
        case 32 * 8 + 2:
            rc = teams ? launch_ws<32, 2, kTeamsF2>(h, in, rm, n, dir32, out, density_only, round_ctr, st)
                       : launch_ws<32, 2>(h, in, rm, n, dir32, out, density_only, round_ctr, st);
            break;
        case 64 * 8 + 4:
            rc = teams && kTeamsF4 ? launch_ws<64, 4, 2>(h, in, rm, n, dir32, out, density_only, round_ctr, st)
                                   : launch_ws<64, 4>(h, in, rm, n, dir32, out, density_only, round_ctr, st);
            break;
        case 32 * 8 + 4: rc = launch_ws<32, 4>(h, in, rm, n, dir32, out, density_only, round_ctr, st); break;
        case 64 * 8 + 2: rc = launch_ws<64, 2>(h, in, rm, n, dir32, out, density_only, round_ctr, st); break;
        case 16 * 8 + 4: rc = launch_ws<16, 4>(h, in, rm, n, dir32, out, density_only, round_ctr, st); break;
        default: return fail(HRT_EINVAL, "unsupported encoding width");
    }
    if (rc) return rc;
    if (timed) {
        CK(cudaEventRecord(h->mev[2 * h->n_timed + 1], st));
        ++h->n_timed;
    }
    ++h->launches;
    return HRT_OK;
}

// sample_batch(p[, d]) on arbitrary device points (probe API + occupancy build).
int field_eval(hrt_handle* h, const double* p, const double* d, int64_t n, float* sigma, float* rgb,
               int32_t* ev, int density_only, int use_occ, int field_frame, cudaStream_t st) {
    if (n == 0) return HRT_OK;
    void *in = nullptr, *dir = nullptr, *res = nullptr, *evb = nullptr;
    CK(cudaMallocAsync(&in, (size_t)n * sizeof(fws::SampleIn), st));
    CK(cudaMallocAsync(&res, (size_t)n * sizeof(float4), st));
    if (d) CK(cudaMallocAsync(&dir, (size_t)n * sizeof(float4), st));
    if (!ev) CK(cudaMallocAsync(&evb, (size_t)n * 4, st));
    int32_t* e = ev ? ev : static_cast<int32_t*>(evb);
    const unsigned g = grid_for(h, n);
    DevField f = h->sc.field;
    kern::k_field_prep<<<g, kThreads, 0, st>>>(f, p, d, n, use_occ, field_frame,
                                               static_cast<fws::SampleIn*>(in),
                                               static_cast<float4*>(dir), e);
    CK(cudaGetLastError());
    int rc = field_ws(h, static_cast<fws::SampleIn*>(in), fws::RowMap{}, n, static_cast<float4*>(dir),
                      static_cast<float4*>(res), density_only, st);
    if (rc == HRT_OK) {
        kern::k_field_post<<<g, kThreads, 0, st>>>(static_cast<float4*>(res), e, n, sigma,
                                                   density_only ? nullptr : rgb);
        CK(cudaGetLastError());
    }
    cudaFreeAsync(in, st);
    cudaFreeAsync(res, st);
    if (dir) cudaFreeAsync(dir, st);
    if (evb) cudaFreeAsync(evb, st);
    return rc;
}

// Occupancy (P4): sigma at every cell centre (field frame) > threshold.
int build_occupancy(hrt_handle* h, double thr) {
    const NeuralField& nf = h->sc.field.nf;
    const int G = nf.occ_res;
    const int64_t n = (int64_t)G * G * G;
    std::vector<double> pts(3 * (size_t)n);
    const DevField& f = h->sc.field;
    for (int z = 0; z < G; ++z)
        for (int y = 0; y < G; ++y)
            for (int x = 0; x < G; ++x) {
                const int64_t c = x + (int64_t)G * (y + (int64_t)G * z);
                const int ijk[3] = {x, y, z};
                for (int a = 0; a < 3; ++a)
                    pts[3 * c + a] = f.lo[a] + ((double)ijk[a] + 0.5) * ((f.hi[a] - f.lo[a]) / G);
            }
    double* dp = nullptr;
    float* ds = nullptr;
    CK(cudaMalloc(&dp, pts.size() * 8));
    CK(cudaMalloc(&ds, (size_t)n * 4));
    CK(cudaMemcpy(dp, pts.data(), pts.size() * 8, cudaMemcpyHostToDevice));
    int rc = field_eval(h, dp, nullptr, n, ds, nullptr, nullptr, 1, 0, 1, 0);
    if (rc == HRT_OK) {
        const int64_t words = (n + 31) / 32;
        kern::k_occ_bits<<<(unsigned)((words + 255) / 256), 256>>>(ds, n, thr, h->occ_dev);
        if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
            rc = fail(HRT_ECUDA, "occupancy build failed");
    }
    cudaFree(dp);
    cudaFree(ds);
    return rc;
}

int ensure_state(hrt_handle* h, int64_t paths) {
    if (paths <= h->cap) return HRT_OK;
    // the old carve is dead from here on: a failed allocation below must not
    // leave a capacity that a later smaller render would trust
    h->cap = 0;
    h->batch_cap = 0;
    if (h->arena) { cudaFree(h->arena); h->arena = nullptr; }
    const int64_t n = paths;
    const int64_t nb = std::min<int64_t>(n * std::max(kern::kRoundSamples, kern::kRoundSamplesSmall), kBatchCap);
    const size_t dbl = (size_t)n * 8, i32 = (size_t)n * 4, f4 = (size_t)n * 16;
    // two passes over the same carve: size it, then assign the pointers
    for (int pass = 0; pass < 2; ++pass) {
        char* base = static_cast<char*>(h->arena);
        size_t off = 0;
        auto take = [&](size_t b) { char* r = base + off; off += (b + 255) & ~size_t(255); return r; };
        auto take_d = [&]() { return reinterpret_cast<double*>(take(dbl)); };
        auto take_i = [&]() { return reinterpret_cast<int32_t*>(take(i32)); };
        PathState& s = h->ps;
        s.ox = take_d(); s.oy = take_d(); s.oz = take_d();
        s.dx = take_d(); s.dy = take_d(); s.dz = take_d();
        s.Lr = take_d(); s.Lg = take_d(); s.Lb = take_d();
        s.Tr = take_d(); s.Tg = take_d(); s.Tb = take_d();
        s.Tm = take_d(); s.t_hit = take_d();
        s.neval = take_i(); s.face = take_i(); s.pix = take_i(); s.smp = take_i();
        s.queue[0] = take_i(); s.queue[1] = take_i();
        kern::MarchState& m = h->ms;
        m.s0 = take_d(); m.delta = take_d();
        m.n = take_i(); m.k = take_i(); m.base = take_i(); m.cnt = take_i();
        m.mq[0] = take_i(); m.mq[1] = take_i();
        m.dir32 = reinterpret_cast<float4*>(take(f4));
        m.h4 = reinterpret_cast<uint64_t*>(take(dbl));
        m.bounce = take_i();
        m.in = reinterpret_cast<fws::SampleIn*>(take((size_t)nb * 16));
        m.sk = reinterpret_cast<int32_t*>(take((size_t)nb * 4));
        m.out = reinterpret_cast<float4*>(take((size_t)nb * 16));
        m.shadow = reinterpret_cast<int32_t*>(take((size_t)nb * 4));
        m.shq = (h->sc.em.n > 0 && kShadowQueue) ? reinterpret_cast<kern::QRay*>(take((size_t)nb * sizeof(kern::QRay)))
                                                 : nullptr;
        s.counters = reinterpret_cast<int32_t*>(take(64 * 4));
        s.stats = reinterpret_cast<unsigned long long*>(take(S_COUNT * 8));
        if (pass == 0) CK(cudaMalloc(&h->arena, off));
    }
    h->cap = n;
    h->batch_cap = nb;
    h->ms.rows_cap = nb;
    h->ms.paths_cap = n;
    return HRT_OK;
}

// Per-bounce ray geometry of the continuous march (grow only): cap paths x
// n_bounces x (7 doubles + 1 int).
int ensure_geo(hrt_handle* h, int32_t n_bounces) {
    const int64_t need = h->cap * std::max(1, n_bounces);
    if (need <= h->geo_n) {
        h->ms.geo.cap = h->cap;
        return HRT_OK;
    }
    h->geo_n = 0;
    if (h->geo_arena) { cudaFree(h->geo_arena); h->geo_arena = nullptr; }
    const size_t dbl = (size_t)need * 8;
    CK(cudaMalloc(&h->geo_arena, 7 * dbl + (size_t)need * 4));
    double* base = static_cast<double*>(h->geo_arena);
    kern::PathGeo& g = h->ms.geo;
    g.ox = base; g.oy = base + need; g.oz = base + 2 * need;
    g.dx = base + 3 * need; g.dy = base + 4 * need; g.dz = base + 5 * need;
    g.t = base + 6 * need;
    g.face = reinterpret_cast<int32_t*>(base + 7 * need);
    g.cap = h->cap;
    h->geo_n = need;
    return HRT_OK;
}

// Persistent host-path buffers (grow only): device pixel list / frame and
// their pinned host staging copies.
int ensure_io(hrt_handle* h, int64_t npx) {
    if (npx <= h->io_cap) return HRT_OK;
    h->io_cap = 0;                       // (stale buffers are never trusted after a failed grow)
    if (h->io_pix) cudaFree(h->io_pix);
    if (h->io_out) cudaFree(h->io_out);
    if (h->io_pix_host) cudaFreeHost(h->io_pix_host);
    if (h->io_out_host) cudaFreeHost(h->io_out_host);
    h->io_pix = nullptr;
    h->io_out = nullptr;
    h->io_pix_host = nullptr;
    h->io_out_host = nullptr;
    const size_t n = (size_t)std::max<int64_t>(npx, 1);
    CK(cudaMalloc(&h->io_pix, n * 4));
    CK(cudaMalloc(&h->io_out, n * 24));
    CK(cudaMallocHost(&h->io_pix_host, n * 4));
    CK(cudaMallocHost(&h->io_out_host, n * 24));
    if (!h->io_stream) CK(cudaStreamCreateWithFlags(&h->io_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : h->io_ev)
        if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->io_cap = npx;
    return HRT_OK;
}

// Is a caller buffer page-locked (then it is DMA'd directly, else staged)?
bool host_pinned(const void* p);

// memcpy split over a few host threads (one core copies ~10 GB/s; the frame
// read-back of the e2e path is 15 MB at 800x800).
void par_copy(char* dst, const char* src, size_t len) {
    constexpr size_t kMin = size_t(1) << 20;
    const int nt = (int)std::min<size_t>(4, std::max<size_t>(1, len / kMin));
    if (nt == 1) { std::memcpy(dst, src, len); return; }
    std::vector<std::thread> ts;
    const size_t part = (len + nt - 1) / nt;
    for (int t = 1; t < nt; ++t) {
        const size_t off = t * part;
        if (off >= len) break;
        ts.emplace_back([=] { std::memcpy(dst + off, src + off, std::min(part, len - off)); });
    }
    std::memcpy(dst, src, std::min(part, len));
    for (auto& t : ts) t.join();
}

bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;               // cudaMallocHost / cudaHostRegister memory
}

int read_counter(hrt_handle* h, int idx, cudaStream_t st, int32_t* v) {
    CK(cudaMemcpyAsync(h->pinned, h->ps.counters + idx, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *v = *h->pinned;
    return HRT_OK;
}

// Samples per path of a march round: kRoundSamples, raised for small (tail)
// rounds so a batch still fills ~kTailTiles 128-row tiles per SM, capped by
// the batch buffer.
#ifndef HRT_TAIL_TILES
#define HRT_TAIL_TILES 8
#endif
constexpr int64_t kTailTiles = HRT_TAIL_TILES;
constexpr int64_t kMaxRoundSamples = 256;      // (k_round_begin uses the same 256)
#ifndef HRT_ROUNDS_PER_CHECK
#define HRT_ROUNDS_PER_CHECK 4
#endif
constexpr int kRoundsPerCheck = HRT_ROUNDS_PER_CHECK;
int32_t round_samples(const hrt_handle* h, int64_t live) {
    int64_t S = kern::kRoundSamples;
    if (kTailTiles > 0) {
        const int64_t want = (int64_t)h->sm_count * 128 * kTailTiles / std::max<int64_t>(live, 1);
        S = std::max<int64_t>(S, std::min<int64_t>(want, kMaxRoundSamples));
    }
    return (int32_t)std::max<int64_t>(1, std::min<int64_t>(S, h->batch_cap / std::max<int64_t>(live, 1)));
}

// ---- stage profiler (hrt_set_profile): pbeg/pend bracket one launch
constexpr int kProfPairs = 4096;

void prof_fold(hrt_handle* h, cudaStream_t st) {
    if (!h->prof || h->pn == 0) return;
    cudaStreamSynchronize(st);
    for (int i = 0; i < h->pn; ++i) {
        float x = 0.f;
        cudaEventElapsedTime(&x, h->pev[2 * i], h->pev[2 * i + 1]);
        h->stage_ms[h->pstage[i]] += x;
    }
    h->pn = 0;
}
// NVTX ranges around every stage's enqueue (named as hrt.h HRT_STAGE_*), so
// an nsys / ncu --nvtx timeline groups the wavefront's launches by stage;
// without an attached tool nvtx3 calls are a null-pointer check.
const char* const kStageName[8] = {"hrt:raygen", "hrt:intersect", "hrt:march_gen", "hrt:field",
                                   "hrt:shadow", "hrt:composite", "hrt:shade", "hrt:accumulate"};
inline void pbeg(hrt_handle* h, cudaStream_t st, int stage) {
    nvtxRangePushA(kStageName[stage]);
    if (h->prof) cudaEventRecord(h->pev[2 * h->pn], st);
}
inline void pend(hrt_handle* h, int stage, cudaStream_t st) {
    nvtxRangePop();
    if (!h->prof) return;
    cudaEventRecord(h->pev[2 * h->pn + 1], st);
    h->pstage[h->pn++] = stage;
    if (h->pn == kProfPairs) prof_fold(h, st);
}

// Queued shadow rays of the round through the blocker tree (persistent).
int shadow_trace(hrt_handle* h, const kern::Args& a, cudaStream_t st) {
    if (!h->ms.shq) return HRT_OK;
    if (h->shadow_blocks == 0) {
        int nb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern::k_shadow_trace, 256, 0));
        h->shadow_blocks = std::max(1, nb) * h->sm_count;
    }
    kern::k_shadow_trace<<<h->shadow_blocks, 256, 0, st>>>(a, h->ms);
    CK(cudaGetLastError());
    ++h->launches;
    return HRT_OK;
}

// NeRF march of every alive path of this bounce: k_seg, then rounds of
// k_gen -> k_field_ws -> k_comp until no path has midpoints left.
int march_neural(hrt_handle* h, const kern::Args& a, int64_t n_paths, cudaStream_t st) {
    const unsigned g = grid_for(h, n_paths);
    const unsigned gs = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_paths + kStepThreads - 1) / kStepThreads,
                                                                         (int64_t)h->sm_count * 16 * 256 / kStepThreads));
    int rc;
    if (!a.trace) {
        // Device-driven fused rounds, no host sync per round:
        //   k_round_begin (queue flip, S, strides) -> k_step (composite the
        //   previous batch + generate the next) -> field engine -> shadows,
        // every kernel reading the round's shape from the device counters.
        // Rounds are enqueued kRoundsPerCheck at a time; the host then checks
        // whether the last round generated any sample (rounds after the end
        // are empty launches).
        pbeg(h, st, HRT_STAGE_MARCH_GEN);
        kern::k_march_begin<<<1, 1, 0, st>>>(h->ps.counters);
        kern::k_seg<<<g, kThreads, 0, st>>>(a, h->ms);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_MARCH_GEN, st);
        h->launches += 2;
        const int32_t target = (int32_t)std::min<int64_t>((int64_t)h->sm_count * 128 * kTailTiles, 1 << 30);
        const int32_t cap = (int32_t)std::min<int64_t>(h->batch_cap, 1 << 30);
        const unsigned gsh = (unsigned)(h->sm_count * 16);
        int32_t round = 0;                       // march round of this chunk
        while (true) {
            for (int k = 0; k < kRoundsPerCheck; ++k, ++round) {
                pbeg(h, st, HRT_STAGE_COMPOSITE);
                kern::k_round_begin<<<1, 1, 0, st>>>(h->ps.counters, h->ps.stats, target, cap,
                                                    h->round_rows, kTimedLaunches);
                if (a.mixed) kern::k_step<true><<<gs, kStepThreads, 0, st>>>(a, h->ms);
                else kern::k_step<false><<<gs, kStepThreads, 0, st>>>(a, h->ms);
                CK(cudaGetLastError());
                pend(h, HRT_STAGE_COMPOSITE, st);
                pbeg(h, st, HRT_STAGE_FIELD);
                // the first rounds carry the L1-coherent primary rays: two encode teams
                if ((rc = field_ws(h, h->ms.in, fws::RowMap{}, 0, h->ms.dir32, h->ms.out, 0, st,
                                   h->ps.counters, round < (h->F == 4 ? kTeamRoundsF4 : kTeamRounds))))
                    return rc;
                pend(h, HRT_STAGE_FIELD, st);
                if (h->sc.em.n > 0) {
                    pbeg(h, st, HRT_STAGE_SHADOW);
                    kern::k_shadow<<<gsh, kThreads, 0, st>>>(a, h->ms, fws::RowMap{}, 0, 1);
                    CK(cudaGetLastError());
                    if ((rc = shadow_trace(h, a, st))) return rc;
                    pend(h, HRT_STAGE_SHADOW, st);
                    ++h->launches;
                }
                h->launches += 2;
                ++h->rounds;
            }
            int32_t ns = 0;
            if ((rc = read_counter(h, C_NS, st, &ns))) return rc;
            if (ns == 0) break;
        }
        return HRT_OK;
    }
    pbeg(h, st, HRT_STAGE_MARCH_GEN);
    kern::k_round_reset<<<1, 1, 0, st>>>(h->ps.counters, 0);
    kern::k_seg<<<g, kThreads, 0, st>>>(a, h->ms);
    CK(cudaGetLastError());
    pend(h, HRT_STAGE_MARCH_GEN, st);
    h->launches += 2;
    int32_t live = 0;
    if ((rc = read_counter(h, C_MQ0, st, &live))) return rc;
    int mc = 0;
    while (live > 0) {
        const int32_t S = round_samples(h, live);
        const unsigned gl = grid_for(h, live);
        pbeg(h, st, HRT_STAGE_MARCH_GEN);
        kern::k_round_reset<<<1, 1, 0, st>>>(h->ps.counters, mc ^ 1);
        kern::k_gen<<<gl, kThreads, 0, st>>>(a, h->ms, mc, S);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_MARCH_GEN, st);
        pbeg(h, st, HRT_STAGE_FIELD);
        if ((rc = field_ws(h, h->ms.in, fws::RowMap{}, (int64_t)live * S, h->ms.dir32, h->ms.out, 0,
                           st)))
            return rc;
        pend(h, HRT_STAGE_FIELD, st);
        if (h->sc.em.n > 0) {
            const int64_t rows = (int64_t)live * S;
            pbeg(h, st, HRT_STAGE_SHADOW);
            kern::k_shadow<<<grid_for(h, rows), kThreads, 0, st>>>(a, h->ms, fws::RowMap{}, rows, 0);
            CK(cudaGetLastError());
            if ((rc = shadow_trace(h, a, st))) return rc;
            pend(h, HRT_STAGE_SHADOW, st);
            ++h->launches;
        }
        pbeg(h, st, HRT_STAGE_COMPOSITE);
        if (a.trace) kern::k_comp<true><<<gl, kThreads, 0, st>>>(a, h->ms, mc);
        else kern::k_comp<false><<<gl, kThreads, 0, st>>>(a, h->ms, mc);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_COMPOSITE, st);
        h->launches += 3;
        ++h->rounds;
        if ((rc = read_counter(h, C_MQ0 + (mc ^ 1), st, &live))) return rc;
        mc ^= 1;
    }
    return HRT_OK;
}

int march(hrt_handle* h, const kern::Args& a, int64_t n_paths, cudaStream_t st) {
    if (h->sc.field.kind == HRT_FIELD_DENSE) {
        pbeg(h, st, HRT_STAGE_COMPOSITE);
        kern::k_march_dense<<<grid_for(h, n_paths), kThreads, 0, st>>>(a);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_COMPOSITE, st);
        ++h->launches;
        return HRT_OK;
    }
    return march_neural(h, a, n_paths, st);
}

// Bounce loop of one chunk (render.py:204-246, or the degenerate tracers
// render.py:249-299 for mode surface / volume).
int run_bounces(hrt_handle* h, kern::Args& a, int64_t paths, int mode, cudaStream_t st) {
    const bool field = h->sc.field.kind != HRT_FIELD_NONE;
    const unsigned g = grid_for(h, paths);
    int rc;
    if (mode == HRT_MODE_VOLUME) {
        a.bounce = 1;
        a.cur = 0;
        a.volume = 1;
        kern::k_reset_queue<<<1, 1, 0, st>>>(h->ps.counters, 1);
        ++h->launches;
        if (field && (rc = march(h, a, paths, st))) return rc;
        return HRT_OK;
    }
    if (h->continuous && field && mode == HRT_MODE_HYBRID && !a.trace &&
        h->sc.field.kind == HRT_FIELD_NEURAL && h->sc.n_bounces >= 1) {
        // continuous wavefront march: bounce 1's rays are intersected here,
        // every later bounce inside the march rounds (kern::advance)
        a.bounce = 1;
        a.cur = 0;
        a.mixed = 1;
        if ((rc = ensure_geo(h, h->sc.n_bounces))) return rc;
        pbeg(h, st, HRT_STAGE_INTERSECT);
        kern::k_reset_queue<<<1, 1, 0, st>>>(h->ps.counters, 1);
        const unsigned gp = (unsigned)std::min<int64_t>((paths + HRT_PATHS_THREADS - 1) / HRT_PATHS_THREADS,
                                                        (int64_t)h->sm_count * 16 * 256 / HRT_PATHS_THREADS);
        if (paths < kCoopPaths) {
            kern::k_paths_coop<<<grid_for(h, paths * 4), kThreads, 0, st>>>(a, h->ms.geo);
        } else if (kPathsByBounce) {
            // bounce-b rays of the paths still going, compacted between launches
            const int32_t* qin = h->ps.queue[0];
            const int32_t* nin = h->ps.counters + C_Q0;
            for (int b = 1; b <= h->sc.n_bounces; ++b) {
                int32_t* qout = h->ms.mq[b & 1];
                int32_t* nout = h->ps.counters + (b & 1 ? C_PB1 : C_PB0);
                kern::k_reset_queue<<<1, 1, 0, st>>>(h->ps.counters, b & 1 ? C_PB1 : C_PB0);
                kern::k_paths_bounce<<<gp, HRT_PATHS_THREADS, 0, st>>>(a, h->ms.geo, b, qin, nin, qout, nout);
                h->launches += 2;
                qin = qout;
                nin = nout;
            }
        } else {
            kern::k_paths<<<gp, HRT_PATHS_THREADS, 0, st>>>(a, h->ms.geo);
        }
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_INTERSECT, st);
        h->launches += 2;
        return march_neural(h, a, paths, st);
    }
    for (int b = 1; b <= h->sc.n_bounces; ++b) {
        a.bounce = b;
        a.cur = (b - 1) & 1;
        pbeg(h, st, HRT_STAGE_INTERSECT);
        kern::k_reset_queue<<<1, 1, 0, st>>>(h->ps.counters, a.cur ^ 1);
        kern::k_intersect<<<g, kThreads, 0, st>>>(a);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_INTERSECT, st);
        if (field && mode == HRT_MODE_HYBRID && (rc = march(h, a, paths, st))) return rc;
        pbeg(h, st, HRT_STAGE_SHADE);
        kern::k_shade<<<g, kThreads, 0, st>>>(a);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_SHADE, st);
        h->launches += 3;
    }
    return HRT_OK;
}

// Shadow entry table (bvh::k_shadow_entry) over a 32^3 world grid around
// the field box, per emitter and light patch; made when the scene has
// emitters and blockers, remade after a blocker refit or a field move.
#ifndef HRT_SHENT_G
#define HRT_SHENT_G 32
#endif
#ifndef HRT_SHENT_P
#define HRT_SHENT_P 8
#endif
constexpr int32_t kShentGrid = HRT_SHENT_G;
int ensure_shadow_entry(hrt_handle* h) {
    DevScene& sc = h->sc;
    const bool want = h->shent_on && HRT_BVH_WIDTH == 4 && sc.em.n > 0 && sc.em.n <= 16 &&
                      sc.blockers.n_faces > 0 && sc.field.kind == HRT_FIELD_NEURAL &&   // (queued shadow rays)
                      h->rfb.n_q < (1 << 23);
    if (!want) {
        sc.shent = nullptr;
        return HRT_OK;
    }
    if (h->shent_ver == h->geo_ver && sc.shent) return HRT_OK;
    const DevField& f = sc.field;
    // world box of the field box (field_from_world is affine: invert its 3x3)
    double lo[3] = {f.lo[0], f.lo[1], f.lo[2]}, hi[3] = {f.hi[0], f.hi[1], f.hi[2]};
    if (!f.identity) {
        const double* m = f.inv;
        const double a = m[0], b = m[1], c = m[2], d = m[4], e = m[5], g = m[6], k = m[8], l = m[9], n = m[10];
        const double det = a * (e * n - g * l) - b * (d * n - g * k) + c * (d * l - e * k);
        if (!(std::fabs(det) > 1e-300)) { sc.shent = nullptr; return HRT_OK; }
        const double R[9] = {(e * n - g * l) / det, (c * l - b * n) / det, (b * g - c * e) / det,
                             (g * k - d * n) / det, (a * n - c * k) / det, (c * d - a * g) / det,
                             (d * l - e * k) / det, (b * k - a * l) / det, (a * e - b * d) / det};
        const double t[3] = {m[3], m[7], m[11]};
        for (int ax = 0; ax < 3; ++ax) { lo[ax] = INFINITY; hi[ax] = -INFINITY; }
        for (int q = 0; q < 8; ++q) {
            const double pf[3] = {(q & 1) ? f.hi[0] : f.lo[0], (q & 2) ? f.hi[1] : f.lo[1],
                                  (q & 4) ? f.hi[2] : f.lo[2]};
            for (int ax = 0; ax < 3; ++ax) {
                double w = 0.0;
                for (int j = 0; j < 3; ++j) w += R[3 * ax + j] * (pf[j] - t[j]);
                lo[ax] = std::min(lo[ax], w);
                hi[ax] = std::max(hi[ax], w);
            }
        }
    }
    const int32_t g = kShentGrid, P = sc.em.n <= 4 ? HRT_SHENT_P : 4;
    d3 glo, cell;
    double inv[3];
    for (int ax = 0; ax < 3; ++ax) {
        const double span = hi[ax] - lo[ax];
        const double pad = 1e-3 * std::max(1.0, span);       // sample points on the box faces fall inside
        const double l0 = lo[ax] - pad, c = (span + 2 * pad) / g;
        (&glo.x)[ax] = l0;
        (&cell.x)[ax] = c;
        inv[ax] = 1.0 / c;
        sc.shent_lo[ax] = l0;
        sc.shent_inv[ax] = inv[ax];
    }
    const int64_t n = (int64_t)g * g * g * sc.em.n * P * P;
    sc.shent = nullptr;                  // (until the new table is complete)
    if (n > h->shent_n) {
        if (h->shent) cudaFree(h->shent);
        h->shent = nullptr;
        h->shent_n = 0;
        CK(cudaMalloc(&h->shent, (size_t)n * 4));
        h->shent_n = n;
    }
    bvh::k_shadow_entry<<<(unsigned)std::min<int64_t>((n + 127) / 128, (int64_t)h->sm_count * 64), 128>>>(
        sc.blockers, sc.em, glo, cell, g, P, h->shent, n);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());         // (renders may run on a non-blocking stream)
    sc.shent = h->shent;
    sc.shent_g = g;
    sc.shent_p = P;
    h->shent_ver = h->geo_ver;
    return HRT_OK;
}

path::Camera to_cam(const hrt_camera& c) {
    path::Camera k{};
    std::memcpy(k.rot, c.rot, sizeof(k.rot));
    std::memcpy(k.pos, c.pos, sizeof(k.pos));
    k.tan_half = c.tan_half;
    k.aspect = c.aspect;
    k.width = c.width;
    k.height = c.height;
    return k;
}

int strat_of(int spp) {
    const int k = (int)std::floor(std::sqrt((double)spp));
    return (k * k == spp && k > 1) ? k : 0;
}

}  // namespace

extern "C" {

const char* hrt_last_error(void) { return g_err.c_str(); }
int hrt_version(void) { return 1; }

int hrt_create(const hrt_scene_desc* d, hrt_handle** out) {
    if (!d || !out) return fail(HRT_EINVAL, "null argument");
    *out = nullptr;
    hrt_handle* h = new hrt_handle();
    auto bail = [&](int rc) { delete h; return rc; };
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    for (cudaEvent_t& e : h->mev) CK(cudaEventCreate(&e));
    CK(cudaMallocHost(&h->pinned, 64));
    {   // keep stream-ordered scratch (probe batches) resident in the pool
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    DevScene& sc = h->sc;
    int rc;
    h->bvh = hrt::build_bvh(d->n_faces, d->v0, d->e1, d->e2);
    h->blk = hrt::build_bvh(d->n_blockers, d->bv0, d->be1, d->be2);
    if ((rc = upload_bvh(h, h->bvh, sc.bvh, h->rf))) return bail(rc);
    if ((rc = upload_bvh(h, h->blk, sc.blockers, h->rfb))) return bail(rc);
    h->mesh_of_host.assign(d->mesh_of, d->mesh_of + d->n_faces);
    for (int32_t m : h->mesh_of_host) h->n_meshes = std::max(h->n_meshes, m + 1);
    if ((rc = setup_refit(h, h->bvh, h->rf))) return bail(rc);
    if ((rc = setup_refit(h, h->blk, h->rfb))) return bail(rc);
    double *normal, *emission;
    int32_t* mesh_of;
    if ((rc = h->upload(d->normal, 3 * (size_t)d->n_faces, &normal))) return bail(rc);
    if ((rc = h->upload(d->emission, 3 * (size_t)d->n_faces, &emission))) return bail(rc);
    if ((rc = h->upload(d->mesh_of, (size_t)d->n_faces, &mesh_of))) return bail(rc);
    sc.normal = normal; sc.emission = emission; sc.mesh_of = mesh_of;
    h->d_normal = normal;
    std::vector<double> r0(std::max(1, d->n_materials));
    for (int m = 0; m < d->n_materials; ++m) {
        const double q = (d->mat_ior[m] - 1.0) / (d->mat_ior[m] + 1.0);
        r0[m] = std::pow(q, 2.0);
    }
    int32_t* mk_;
    double *mrgb, *mior, *mr0;
    if ((rc = h->upload(d->mat_kind, (size_t)d->n_materials, &mk_))) return bail(rc);
    if ((rc = h->upload(d->mat_rgb, 3 * (size_t)d->n_materials, &mrgb))) return bail(rc);
    if ((rc = h->upload(d->mat_ior, (size_t)d->n_materials, &mior))) return bail(rc);
    if ((rc = h->upload(r0.data(), (size_t)d->n_materials, &mr0))) return bail(rc);
    sc.mat = {mk_, mrgb, mior, mr0};
    sc.em.n = d->n_emitters;
    double *et, *ec, *er;
    if ((rc = h->upload(d->emitter_tris, 9 * (size_t)d->n_emitters, &et))) return bail(rc);
    if ((rc = h->upload(d->emitter_cdf, (size_t)d->n_emitters, &ec))) return bail(rc);
    if ((rc = h->upload(d->emitter_rsrc, (size_t)d->n_emitters, &er))) return bail(rc);
    sc.em.tris = et; sc.em.cdf = ec; sc.em.r_src = er;
    if ((rc = setup_field(h, d->field))) return bail(rc);
    sc.n_bounces = d->n_bounces;
    sc.threshold = d->threshold;
    sc.march_step = d->march_step;
    sc.spawn_eps = d->spawn_eps;
    sc.sample_cap = d->sample_cap;
    sc.early_t = d->early_t;
    if (!(d->march_step > 0)) return bail(fail(HRT_EINVAL, "march step must be > 0"));
    if (d->field.kind == HRT_FIELD_NEURAL && !d->field.occ_bits) {
        if ((rc = build_occupancy(h, d->field.occ_threshold))) return bail(rc);
    }
    if ((rc = h->alloc((size_t)kTimedLaunches * 16, reinterpret_cast<void**>(&h->round_rows)))) return bail(rc);
    {
        const char* e = std::getenv("HRT_SHADOW_ENTRY");
        h->shent_on = !(e && e[0] == '0');
    }
    CK(cudaDeviceSynchronize());
    *out = h;
    return HRT_OK;
}

int hrt_destroy(hrt_handle* h) {
    delete h;
    return HRT_OK;
}

int hrt_set_trace(hrt_handle* h, int32_t* records, int64_t cap) {
    if (!h) return fail(HRT_EINVAL, "null handle");
    h->trace = records;
    h->trace_cap = cap;
    return HRT_OK;
}

int hrt_set_march(hrt_handle* h, int32_t continuous) {
    if (!h) return fail(HRT_EINVAL, "null handle");
    h->continuous = continuous != 0;
    return HRT_OK;
}

int hrt_set_config(hrt_handle* h, int32_t n_bounces, double threshold, double march_step,
                   double spawn_eps, int32_t sample_cap, double early_t) {
    if (!h) return fail(HRT_EINVAL, "null handle");
    if (!(march_step > 0)) return fail(HRT_EINVAL, "march step must be > 0");
    if (n_bounces < 0) return fail(HRT_EINVAL, "n_bounces must be >= 0");
    DevScene& sc = h->sc;
    sc.n_bounces = n_bounces;
    sc.threshold = threshold;
    sc.march_step = march_step;
    sc.spawn_eps = spawn_eps;
    sc.sample_cap = sample_cap;
    sc.early_t = early_t;
    return HRT_OK;
}

int hrt_set_profile(hrt_handle* h, int32_t on) {
    if (!h) return fail(HRT_EINVAL, "null handle");
    if (on && h->pev.empty()) {
        h->pev.resize(2 * kProfPairs);
        h->pstage.resize(kProfPairs);
        for (cudaEvent_t& e : h->pev) CK(cudaEventCreate(&e));
    }
    h->prof = on != 0;
    return HRT_OK;
}

int hrt_render(hrt_handle* h, const hrt_camera* cam, int32_t spp, uint64_t seed, int32_t mode,
               const int32_t* pixels, int64_t n_pixels, double* out, hrt_stats* stats, void* stream) {
    if (!h || !cam) return fail(HRT_EINVAL, "null argument");
    if (spp < 1) return fail(HRT_EINVAL, "spp must be >= 1");
    const int32_t by_pixel = (mode & HRT_OUT_BY_PIXEL) ? 1 : 0;
    mode &= ~HRT_OUT_BY_PIXEL;
    if (mode < 0 || mode > 2) return fail(HRT_EINVAL, "bad mode");
    if (cam->width < 1 || cam->height < 1) return fail(HRT_EINVAL, "bad resolution");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t total_pix = pixels ? n_pixels : (int64_t)cam->width * cam->height;
    if (pixels && total_pix <= 0) {            // empty pixel list (e.g. a rank without tiles)
        if (stats) *stats = hrt_stats{};
        return HRT_OK;
    }
    if (!out) return fail(HRT_EINVAL, "null argument");
    const int64_t chunk_pix = std::max<int64_t>(1, (h->F == 4 ? kMaxPathsF4 : kMaxPaths) / spp);
    int rc;
    if ((rc = ensure_state(h, std::min<int64_t>(total_pix, chunk_pix) * spp))) return rc;
    if ((rc = ensure_shadow_entry(h))) return rc;
    CK(cudaMemsetAsync(h->ps.counters, 0, 64 * 4, st));
    CK(cudaMemsetAsync(h->ps.stats, 0, S_COUNT * 8, st));
    h->n_timed = 0;
    h->launches = 0;
    h->rounds = 0;
    h->batch_rows = 0;
    h->pn = 0;
    for (double& x : h->stage_ms) x = 0.0;
    CK(cudaEventRecord(h->ev0, st));
    for (int64_t p0 = 0; p0 < total_pix; p0 += chunk_pix) {
        const int64_t np = std::min(chunk_pix, total_pix - p0);
        const int64_t paths = np * spp;
        kern::Args a{};
        a.sc = h->sc;
        a.ps = h->ps;
        a.cam = to_cam(*cam);
        a.pixels = pixels ? pixels + p0 : nullptr;
        a.pixel_base = pixels ? 0 : p0;
        a.n_slots = np;
        a.spp = spp;
        a.strat = strat_of(spp);
        a.seed = seed;
        a.out = out;
        a.out_offset = p0;
        a.tiled = (!pixels && kTiledFrame) ? 1 : 0;
        a.out_by_pixel = by_pixel;
        a.trace = h->trace;
        a.trace_cap = h->trace_cap;
        pbeg(h, st, HRT_STAGE_RAYGEN);
        kern::k_raygen<<<grid_for(h, paths), kThreads, 0, st>>>(a);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_RAYGEN, st);
        h->launches += 2;   // raygen + accumulate
        if ((rc = run_bounces(h, a, paths, mode, st))) return rc;
        pbeg(h, st, HRT_STAGE_ACCUMULATE);
        kern::k_accumulate<<<grid_for(h, np), kThreads, 0, st>>>(a);
        CK(cudaGetLastError());
        pend(h, HRT_STAGE_ACCUMULATE, st);
    }
    prof_fold(h, st);
    CK(cudaEventRecord(h->ev1, st));
    h->trace = nullptr;
    int32_t ctr[64];
    unsigned long long tot[S_COUNT];
    CK(cudaMemcpyAsync(ctr, h->ps.counters, sizeof(ctr), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(tot, h->ps.stats, sizeof(tot), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (stats) {
        stats->paths = total_pix * spp;
        stats->nerf_samples = (int64_t)tot[S_SAMPLES];
        stats->shadow_rays = (int64_t)tot[S_SHADOW_USED];
        stats->shadow_traced = (int64_t)tot[S_SHADOW];
        stats->bounce_rays = (int64_t)tot[S_SEGMENTS];
        stats->trace_records = ctr[C_TRACE];
        stats->evaluated = (int64_t)tot[S_EVALS];
        stats->rounds = h->rounds;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev0, h->ev1);
        stats->ms = ms;
        float mms = 0.f;
        for (int i = 0; i < h->n_timed; ++i) {
            float x = 0.f;
            cudaEventElapsedTime(&x, h->mev[2 * i], h->mev[2 * i + 1]);
            mms += x;
        }
        stats->field_ms = mms;
        stats->field_launches = h->n_timed;
        stats->launches = h->launches;
        for (int i = 0; i < 8; ++i) stats->stage_ms[i] = (float)h->stage_ms[i];
        stats->batch_rows = h->batch_rows + (int64_t)tot[S_ROWS];
        h->n_round_rows = std::min<int32_t>(ctr[C_RIDX], kTimedLaunches);
#ifdef HRT_COUNT_STEPS
        fprintf(stderr, "shadow trace: cast %llu traced %llu blocked %llu | steps %llu, of blocked rays %llu\n",
                tot[S_SHADOW], tot[9], tot[7], tot[5], tot[6]);
#endif
    }
    if (ctr[C_NONFINITE] != 0) return fail(HRT_ENONFINITE, "non-finite or negative radiance in frame");
    return HRT_OK;
}

int hrt_transport(hrt_handle* h, const hrt_camera* cams, int32_t n_poses, int32_t spp, uint64_t seed,
                  int32_t max_depth, double* out, void* stream) {
    if (!h || !cams || !out) return fail(HRT_EINVAL, "null argument");
    if (n_poses < 1 || spp < 1 || max_depth < 1) return fail(HRT_EINVAL, "n_poses, spp, max_depth must be >= 1");
    if (h->sc.field.kind != HRT_FIELD_NONE) return fail(HRT_EINVAL, "estimation scenes must not contain a radiance field");
    const int32_t w = cams[0].width, hh = cams[0].height;
    for (int i = 0; i < n_poses; ++i)
        if (cams[i].width != w || cams[i].height != hh) return fail(HRT_EINVAL, "all poses must share one resolution");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t npix = (int64_t)w * hh;
    const int32_t F = h->bvh.n_faces;
    const int32_t per_batch = (int32_t)std::max<int64_t>(1, 65536 / npix);   // emitters.py:151
    CK(cudaMemsetAsync(out, 0, (size_t)n_poses * npix * F * 3 * sizeof(double), st));
    const int64_t chunk_pix = std::max<int64_t>(1, kMaxPaths / spp);
    int rc;
    if ((rc = ensure_state(h, std::min<int64_t>(npix, chunk_pix) * spp))) return rc;
    if ((rc = ensure_shadow_entry(h))) return rc;
    const int64_t nrec = std::min<int64_t>(npix, chunk_pix) * spp * max_depth;
    int32_t* rface = nullptr;
    double* rval = nullptr;
    CK(cudaMallocAsync(&rface, (size_t)nrec * 4, st));
    CK(cudaMallocAsync(&rval, (size_t)nrec * 24, st));
    DevScene sc = h->sc;
    sc.n_bounces = max_depth;                     // emitters.py:140 (temporary n_bounces)
    for (int pose = 0; pose < n_poses && rc == HRT_OK; ++pose) {
        for (int64_t p0 = 0; p0 < npix; p0 += chunk_pix) {
            const int64_t np = std::min(chunk_pix, npix - p0), paths = np * spp;
            kern::Args a{};
            a.sc = sc;
            a.ps = h->ps;
            a.cam = to_cam(cams[pose]);
            a.pixel_base = p0;
            a.n_slots = np;
            a.spp = spp;
            a.strat = strat_of(spp);
            a.seed = seed;
            a.tiled = 0;
            CK(cudaMemsetAsync(rface, 0xff, (size_t)paths * max_depth * 4, st));
            CK(cudaMemsetAsync(h->ps.counters, 0, 64 * 4, st));
            kern::k_raygen<<<grid_for(h, paths), kThreads, 0, st>>>(a);
            CK(cudaGetLastError());
            const unsigned g = grid_for(h, paths);
            for (int b = 1; b <= max_depth; ++b) {
                a.bounce = b;
                a.cur = (b - 1) & 1;
                kern::k_reset_queue<<<1, 1, 0, st>>>(h->ps.counters, a.cur ^ 1);
                kern::k_intersect<<<g, kThreads, 0, st>>>(a);
                kern::k_shade_transport<<<g, kThreads, 0, st>>>(a, max_depth, rface, rval);
                CK(cudaGetLastError());
            }
            kern::k_transport_reduce<<<grid_for(h, np), kThreads, 0, st>>>(
                np, spp, max_depth, per_batch, F, rface, rval, (int64_t)pose * npix + p0, out);
            CK(cudaGetLastError());
        }
    }
    CK(cudaFreeAsync(rface, st));
    CK(cudaFreeAsync(rval, st));
    CK(cudaStreamSynchronize(st));
    return rc;
}

int hrt_trace_paths(hrt_handle* h, const double* o, const double* d, const int64_t* pixel,
                    const int64_t* sample, int64_t n, uint64_t seed, int32_t mode, double* L,
                    void* stream) {
    if (!h || (n > 0 && (!o || !d || !pixel || !sample || !L))) return fail(HRT_EINVAL, "null argument");
    if (mode < 0 || mode > 2) return fail(HRT_EINVAL, "bad mode");
    if (n > kMaxPaths) return fail(HRT_EINVAL, "too many paths for one call");
    if (n == 0) return HRT_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc;
    if ((rc = ensure_state(h, n))) return rc;
    if ((rc = ensure_shadow_entry(h))) return rc;
    CK(cudaMemsetAsync(h->ps.counters, 0, 64 * 4, st));
    CK(cudaMemsetAsync(h->ps.stats, 0, S_COUNT * 8, st));
    kern::Args a{};
    a.sc = h->sc;
    a.ps = h->ps;
    a.n_slots = n;
    a.spp = 1;
    a.seed = seed;
    kern::k_load_rays<<<grid_for(h, n), kThreads, 0, st>>>(a, o, d, pixel, sample);
    CK(cudaGetLastError());
    if ((rc = run_bounces(h, a, n, mode, st))) return rc;
    kern::k_gather_L<<<grid_for(h, n), kThreads, 0, st>>>(a, L);
    CK(cudaGetLastError());
    int32_t ctr[64];
    CK(cudaMemcpyAsync(ctr, h->ps.counters, sizeof(ctr), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (ctr[C_NONFINITE] != 0) return fail(HRT_ENONFINITE, "NaN radiance in path batch");
    return HRT_OK;
}

int hrt_render_host(hrt_handle* h, const hrt_camera* cam, int32_t spp, uint64_t seed, int32_t mode,
                    const int32_t* pixels, int64_t n_pixels, double* out, hrt_stats* stats) {
    if (!h || !cam || !out) return fail(HRT_EINVAL, "null argument");
    const int64_t npx = pixels ? n_pixels : (int64_t)cam->width * cam->height;
    int rc;
    if ((rc = ensure_io(h, npx))) return rc;
    cudaStream_t st = h->io_stream;
    const size_t in_bytes = (size_t)npx * 4, out_bytes = (size_t)npx * 24;
    // page-locked caller buffers are DMA'd directly; pageable ones are staged
    // through the handle's pinned buffers
    const bool in_direct = pixels && host_pinned(pixels);
    const bool out_direct = host_pinned(out);
    if (pixels) {
        if (in_direct) {
            CK(cudaMemcpyAsync(h->io_pix, pixels, in_bytes, cudaMemcpyHostToDevice, st));
        } else {
            par_copy(reinterpret_cast<char*>(h->io_pix_host), reinterpret_cast<const char*>(pixels), in_bytes);
            CK(cudaMemcpyAsync(h->io_pix, h->io_pix_host, in_bytes, cudaMemcpyHostToDevice, st));
        }
    }
    rc = hrt_render(h, cam, spp, seed, mode, pixels ? h->io_pix : nullptr, npx, h->io_out, stats, st);
    if (rc == HRT_OK || rc == HRT_ENONFINITE) {
        if (out_direct) {
            CK(cudaMemcpyAsync(out, h->io_out, out_bytes, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            return rc;
        }
        // staging: the frame comes back in kIoChunks DMA pieces; the pinned ->
        // caller copy of piece k overlaps the DMA of pieces k+1..
        const size_t piece = (out_bytes / kIoChunks + 4095) & ~size_t(4095);
        int nk = 0;
        for (size_t off = 0; off < out_bytes; off += piece, ++nk) {
            const size_t len = std::min(piece, out_bytes - off);
            CK(cudaMemcpyAsync(reinterpret_cast<char*>(h->io_out_host) + off,
                               reinterpret_cast<const char*>(h->io_out) + off, len, cudaMemcpyDeviceToHost, st));
            CK(cudaEventRecord(h->io_ev[nk], st));
        }
        for (int k = 0; k < nk; ++k) {
            CK(cudaEventSynchronize(h->io_ev[k]));
            const size_t off = (size_t)k * piece, len = std::min(piece, out_bytes - off);
            par_copy(reinterpret_cast<char*>(out) + off, reinterpret_cast<const char*>(h->io_out_host) + off, len);
        }
    }
    return rc;
}

int hrt_refit(hrt_handle* h, const double* v0, const double* e1, const double* e2, const double* normal,
              const double* bv0, const double* be1, const double* be2) {
    if (!h) return fail(HRT_EINVAL, "null handle");
    int rc;
    if (h->bvh.n_faces && v0 && e1 && e2) {
        if ((rc = refit_gpu(h, h->bvh, h->rf, h->sc.bvh, v0, e1, e2))) return rc;
        if (normal)
            CK(cudaMemcpy(h->d_normal, normal, 3 * (size_t)h->bvh.n_faces * 8, cudaMemcpyHostToDevice));
    }
    if (h->blk.n_faces && bv0 && be1 && be2) {
        if ((rc = refit_gpu(h, h->blk, h->rfb, h->sc.blockers, bv0, be1, be2))) return rc;
        h->blk_stale = false;
    }
    CK(cudaDeviceSynchronize());
    return HRT_OK;
}

// Rebuild a tree as a forest of per-mesh trees (group = mesh of each face in
// this tree's face order), re-upload it and its refit state.
int to_forest(hrt_handle* h, hrt::BvhHost& b, RefitState& r, DevBvh& dev, const std::vector<int32_t>& group) {
    const int32_t n = b.n_faces;
    if (n == 0) return HRT_OK;
    std::vector<double> v0(3 * (size_t)n), e1(3 * (size_t)n), e2(3 * (size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        const int32_t f = b.tri_id[i];
        std::memcpy(&v0[3 * (size_t)f], &b.tri[9 * (size_t)i], 24);
        std::memcpy(&e1[3 * (size_t)f], &b.tri[9 * (size_t)i + 3], 24);
        std::memcpy(&e2[3 * (size_t)f], &b.tri[9 * (size_t)i + 6], 24);
    }
    std::vector<int32_t> begin;
    for (int32_t f = 0; f < n; ++f)
        if (f == 0 || group[f] != group[f - 1]) begin.push_back(f);
    begin.push_back(n);
    if (begin.size() < 3) return HRT_OK;              // one mesh: the tree already refits tightly
    b = hrt::build_forest(n, v0.data(), e1.data(), e2.data(), begin);
    int rc;
    if ((rc = upload_bvh(h, b, dev, r))) return rc;
    return setup_refit(h, b, r);
}

int hrt_set_rigid_base(hrt_handle* h, const double* corners, const int32_t* blocker_faces) {
    if (!h || (h->bvh.n_faces && !corners)) return fail(HRT_EINVAL, "null argument");
    if (h->blk.n_faces && !blocker_faces) return fail(HRT_EINVAL, "blocker face map required");
    int rc;
    if (h->rf.roots.empty() && h->rfb.roots.empty()) {
        // rigid meshes: one tree per mesh + a per-frame top level, so refits stay tight
        if ((rc = to_forest(h, h->bvh, h->rf, h->sc.bvh, h->mesh_of_host))) return rc;
        std::vector<int32_t> bg(h->blk.n_faces);
        for (int32_t i = 0; i < h->blk.n_faces; ++i) bg[i] = h->mesh_of_host[blocker_faces[i]];
        if ((rc = to_forest(h, h->blk, h->rfb, h->sc.blockers, bg))) return rc;
    }
    if (!h->rigid_base) {
        if ((rc = h->alloc((size_t)std::max(1, h->bvh.n_faces) * 9 * 8, reinterpret_cast<void**>(&h->rigid_base))))
            return rc;
        if ((rc = h->alloc((size_t)std::max(1, h->blk.n_faces) * 4, reinterpret_cast<void**>(&h->blk_map))))
            return rc;
    }
    CK(cudaMemcpy(h->rigid_base, corners, (size_t)h->bvh.n_faces * 9 * 8, cudaMemcpyHostToDevice));
    if (h->blk.n_faces)
        CK(cudaMemcpy(h->blk_map, blocker_faces, (size_t)h->blk.n_faces * 4, cudaMemcpyHostToDevice));
    return HRT_OK;
}

// Blocker forest refit from the current rigid-moved faces (hrt_refit_rigid).
static int ensure_blockers(hrt_handle* h) {
    if (!h->blk_stale) return HRT_OK;
    const int32_t n = h->bvh.n_faces, nb = h->blk.n_faces;
    const unsigned gb = (unsigned)std::min<int64_t>((nb + 255) / 256, 148 * 16);
    bvh::k_gather_faces<<<gb, 256>>>(h->rf.src, n, h->blk_map, nb, h->rfb.src);
    CK(cudaGetLastError());
    const int rc = refit_from_src(h, h->blk, h->rfb, h->sc.blockers);
    if (rc == HRT_OK) h->blk_stale = false;
    return rc;
}

int hrt_refit_rigid(hrt_handle* h, const double* xf, int32_t n_meshes) {
    if (!h || !xf) return fail(HRT_EINVAL, "null argument");
    if (!h->rigid_base) return fail(HRT_EINVAL, "hrt_set_rigid_base first");
    if (h->bvh.n_faces == 0) return HRT_OK;
    if (n_meshes != h->n_meshes) return fail(HRT_EINVAL, "refit_rigid: one 3x4 transform per mesh required");
    if (n_meshes > h->rigid_xf_cap) {            // persistent transform buffer (grow only)
        h->rigid_xf_cap = 0;
        if (h->rigid_xf) cudaFree(h->rigid_xf);
        h->rigid_xf = nullptr;
        CK(cudaMalloc(&h->rigid_xf, (size_t)n_meshes * 12 * 8));
        h->rigid_xf_cap = n_meshes;
    }
    double* dxf = h->rigid_xf;
    CK(cudaMemcpy(dxf, xf, (size_t)n_meshes * 12 * 8, cudaMemcpyHostToDevice));
    const int32_t n = h->bvh.n_faces;
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    bvh::k_rigid_faces<<<g, 256>>>(h->rigid_base, h->sc.mesh_of, dxf, n_meshes, n, h->rf.src, h->d_normal);
    CK(cudaGetLastError());
    int rc = refit_from_src(h, h->bvh, h->rf, h->sc.bvh);
    // the shadow-blocker forest is only traversed by shadow rays: without
    // emitters its refit waits until something queries it (hrt_intersect)
    if (rc == HRT_OK && h->blk.n_faces) {
        h->blk_stale = true;
        if (h->sc.em.n > 0) rc = ensure_blockers(h);
    }
    CK(cudaDeviceSynchronize());
    return rc;
}

int hrt_field_sample(hrt_handle* h, const double* points, const double* dirs, int64_t n, float* sigma,
                     float* rgb, int32_t* evaluated, int32_t use_occupancy, void* stream) {
    if (!h || (n > 0 && (!points || !sigma))) return fail(HRT_EINVAL, "null argument");
    if (h->sc.field.kind != HRT_FIELD_NEURAL) return fail(HRT_EINVAL, "scene has no neural field");
    if (dirs && !rgb) return fail(HRT_EINVAL, "rgb output required with dirs");
    return field_eval(h, points, dirs, n, sigma, rgb, evaluated, dirs ? 0 : 1, use_occupancy, 0,
                      static_cast<cudaStream_t>(stream));
}

int hrt_field_encode(hrt_handle* h, const double* points, int64_t n, float* features, uint32_t* indices,
                     void* stream) {
    if (!h || (n > 0 && (!points || !features))) return fail(HRT_EINVAL, "null argument");
    if (h->sc.field.kind != HRT_FIELD_NEURAL) return fail(HRT_EINVAL, "scene has no neural field");
    if (n == 0) return HRT_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned g = grid_for(h, n);
    const DevField& f = h->sc.field;
    switch (h->E * 8 + h->F) {
        case 16 * 8 + 2: kern::k_field_encode<16, 2><<<g, kThreads, 0, st>>>(f, points, n, features, indices); break;
        case 32 * 8 + 2: kern::k_field_encode<32, 2><<<g, kThreads, 0, st>>>(f, points, n, features, indices); break;
        case 64 * 8 + 4: kern::k_field_encode<64, 4><<<g, kThreads, 0, st>>>(f, points, n, features, indices); break;
        case 32 * 8 + 4: kern::k_field_encode<32, 4><<<g, kThreads, 0, st>>>(f, points, n, features, indices); break;
        case 64 * 8 + 2: kern::k_field_encode<64, 2><<<g, kThreads, 0, st>>>(f, points, n, features, indices); break;
        case 16 * 8 + 4: kern::k_field_encode<16, 4><<<g, kThreads, 0, st>>>(f, points, n, features, indices); break;
        default: return fail(HRT_EINVAL, "unsupported encoding width");
    }
    CK(cudaGetLastError());
    return HRT_OK;
}

int hrt_occupancy(hrt_handle* h, uint32_t* host_words, int64_t n_words) {
    if (!h || !host_words) return fail(HRT_EINVAL, "null argument");
    if (h->sc.field.kind != HRT_FIELD_NEURAL) return fail(HRT_EINVAL, "scene has no neural field");
    if (n_words < h->occ_words) return fail(HRT_EINVAL, "buffer too small");
    CK(cudaMemcpy(host_words, h->occ_dev, (size_t)h->occ_words * 4, cudaMemcpyDeviceToHost));
    return HRT_OK;
}

int hrt_intersect(hrt_handle* h, int32_t blocker, int32_t any, const double* o, const double* d,
                  const double* t_min, const double* t_max, int64_t n, double* t, int64_t* face,
                  uint8_t* hit, void* stream) {
    if (!h || (n > 0 && (!o || !d))) return fail(HRT_EINVAL, "null argument");
    if (any ? !hit : (!t || !face)) return fail(HRT_EINVAL, "missing output");
    if (n == 0) return HRT_OK;
    if (blocker) {
        int rc;
        if ((rc = ensure_blockers(h))) return rc;
    }
    const DevBvh& b = blocker ? h->sc.blockers : h->sc.bvh;
    kern::k_rays<<<grid_for(h, n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        b, o, d, t_min, t_max, n, any, t, face, hit);
    CK(cudaGetLastError());
    return HRT_OK;
}

int hrt_uniform(const int64_t* keys, int64_t n, double* out, void* stream) {
    if (n > 0 && (!keys || !out)) return fail(HRT_EINVAL, "null argument");
    if (n == 0) return HRT_OK;
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    kern::k_uniform<<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(keys, n, out);
    CK(cudaGetLastError());
    return HRT_OK;
}

int hrt_primary_rays(const hrt_camera* cam, const int64_t* pixel, const int64_t* sample, int64_t n,
                     uint64_t seed, int32_t spp, double* o, double* d, void* stream) {
    if (!cam || (n > 0 && (!pixel || !sample || !o || !d))) return fail(HRT_EINVAL, "null argument");
    if (spp < 1) return fail(HRT_EINVAL, "spp must be >= 1");
    if (n == 0) return HRT_OK;
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    kern::k_primary<<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(to_cam(*cam), pixel, sample, n, seed,
                                                                      strat_of(spp), o, d);
    CK(cudaGetLastError());
    return HRT_OK;
}

int hrt_finalize(int32_t width, int32_t height, const double* src, const int32_t* pixel, int64_t n,
                 int32_t hdr, uint8_t* out, int64_t cap, int64_t* nbytes, void* stream) {
    if (width < 1 || height < 1 || !nbytes || (n > 0 && !src)) return fail(HRT_EINVAL, "bad arguments");
    if (!pixel && n != (int64_t)width * height) return fail(HRT_EINVAL, "raster source needs w*h rows");
    char head[64];
    const int hl = hdr ? std::snprintf(head, sizeof(head), "PF\n%d %d\n-1.0\n", width, height)
                       : std::snprintf(head, sizeof(head), "P6\n%d %d\n255\n", width, height);
    const int64_t total = hl + (int64_t)width * height * 3 * (hdr ? 4 : 1);
    *nbytes = total;
    if (!out) return HRT_OK;                         // size query
    if (cap < total) return fail(HRT_EINVAL, "output buffer too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t* bad = nullptr;
    CK(cudaMallocAsync(&bad, 4, st));
    CK(cudaMemsetAsync(bad, 0, 4, st));
    CK(cudaMemcpyAsync(out, head, hl, cudaMemcpyHostToDevice, st));
    if (n > 0) {
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
        fin::k_finalize<<<g, 256, 0, st>>>(width, height, src, pixel, n, hdr, hl, out, bad);
        CK(cudaGetLastError());
    }
    int32_t nb = 0;
    CK(cudaMemcpyAsync(&nb, bad, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(bad, st));
    CK(cudaStreamSynchronize(st));
    if (nb) return fail(HRT_ENONFINITE, "finalize requires finite radiance");
    return HRT_OK;
}

int hrt_buffer_alloc(int64_t bytes, void** ptr) {
    if (!ptr || bytes <= 0) return fail(HRT_EINVAL, "bad arguments");
    CK(cudaMalloc(ptr, (size_t)bytes));
    return HRT_OK;
}

int hrt_buffer_free(void* ptr) {
    if (ptr) CK(cudaFree(ptr));
    return HRT_OK;
}

int hrt_ipc_handle(const void* ptr, uint8_t* handle64) {
    if (!ptr || !handle64) return fail(HRT_EINVAL, "null argument");
    cudaIpcMemHandle_t hd;
    CK(cudaIpcGetMemHandle(&hd, const_cast<void*>(ptr)));
    static_assert(sizeof(hd) == 64, "ipc handle size");
    std::memcpy(handle64, &hd, 64);
    return HRT_OK;
}

int hrt_ipc_open(const uint8_t* handle64, void** ptr) {
    if (!ptr || !handle64) return fail(HRT_EINVAL, "null argument");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle64, 64);
    CK(cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    return HRT_OK;
}

int hrt_ipc_close(void* ptr) {
    if (ptr) CK(cudaIpcCloseMemHandle(ptr));
    return HRT_OK;
}

int hrt_gather_peak(hrt_handle* h, int32_t mode, double* gbs) {
    if (!h || !gbs) return fail(HRT_EINVAL, "null argument");
    if (h->sc.field.kind != HRT_FIELD_NEURAL || (h->F != 2 && h->F != 4))
        return fail(HRT_EINVAL, "needs a neural field (F = 2 or 4)");
    if (mode < 0 || mode > 2) return fail(HRT_EINVAL, "mode: 0 LSU, 1 TEX, 2 both");
    const NeuralField& nf = h->sc.field.nf;
    // an L2-resident window (<= 64 MiB) of the table: the probe measures the L1-miss request
    // ceiling to L2, not DRAM (cfg4's 344 MiB table would make it a DRAM random-read probe)
    const uint32_t n = (uint32_t)std::min<int64_t>(h->tab_entries, (int64_t(64) << 20) / (4 * h->F));
    float* sink = nullptr;
    CK(cudaMalloc(&sink, 4));
    const int threads = 512, blocks = h->sm_count * 4, iters = 64;
    const float2* tab2 = reinterpret_cast<const float2*>(nf.table);
    const float4* tab4 = reinterpret_cast<const float4*>(nf.table);
    const bool f4 = h->F == 4;
    cudaStream_t s2 = nullptr;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    auto launch = [&](cudaStream_t st, bool tex) {
        if (f4 && tex) probe::k_gather<true><<<blocks, threads, 0, st>>>(tab4, nf.tex, n, iters, sink);
        else if (f4) probe::k_gather<false><<<blocks, threads, 0, st>>>(tab4, nf.tex, n, iters, sink);
        else if (tex) probe::k_gather<true><<<blocks, threads, 0, st>>>(tab2, nf.tex, n, iters, sink);
        else probe::k_gather<false><<<blocks, threads, 0, st>>>(tab2, nf.tex, n, iters, sink);
    };
    auto run = [&]() {       // mode 2: LSU and TEX kernels side by side on two streams
        if (mode == 2) {
            CK(cudaEventRecord(h->ev0, 0));
            CK(cudaStreamWaitEvent(s2, h->ev0, 0));
            launch(0, false);
            launch(s2, true);
            CK(cudaEventRecord(h->ev1, s2));
            CK(cudaStreamWaitEvent(0, h->ev1, 0));
        } else {
            launch(0, mode == 1);
        }
        return HRT_OK;
    };
    int rc;
    if ((rc = run())) return rc;                       // warm (table into L2)
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, 0));
    const int reps = 5;
    for (int i = 0; i < reps; ++i)
        if ((rc = run())) return rc;
    CK(cudaEventRecord(e1, 0));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double loads = (double)blocks * threads * iters * 8 * reps * (mode == 2 ? 2 : 1);
    *gbs = loads * (f4 ? 16.0 : 8.0) / (ms * 1e-3) / 1e9;   // useful bytes: one entry per gather
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s2);
    cudaFree(sink);
    return HRT_OK;
}

int hrt_round_rows(hrt_handle* h, int64_t* rows, int64_t* samples, float* field_ms, int32_t cap, int32_t* n) {
    if (!h || !n) return fail(HRT_EINVAL, "null argument");
    // device-driven rounds of the last hrt_render: round i launched the render's i-th
    // field-engine pass (timed by the mev events in launch order)
    const int32_t m = std::min(h->n_round_rows, std::min(cap, h->n_timed));
    *n = m;
    if (m <= 0) return HRT_OK;
    if (rows) CK(cudaMemcpy(rows, h->round_rows, (size_t)m * 8, cudaMemcpyDeviceToHost));
    if (samples) {               // cumulative snapshots at each round's start -> per-round counts
        std::vector<int64_t> snap(m);
        CK(cudaMemcpy(snap.data(), h->round_rows + kTimedLaunches, (size_t)m * 8, cudaMemcpyDeviceToHost));
        unsigned long long tot[S_COUNT];
        CK(cudaMemcpy(tot, h->ps.stats, sizeof(tot), cudaMemcpyDeviceToHost));
        for (int32_t i = 0; i < m; ++i)
            samples[i] = (i + 1 < m ? snap[i + 1] : (int64_t)tot[S_EVALS]) - snap[i];
    }
    if (field_ms) {
        for (int32_t i = 0; i < m; ++i) {
            float x = 0.f;
            cudaEventElapsedTime(&x, h->mev[2 * i], h->mev[2 * i + 1]);
            field_ms[i] = x;
        }
    }
    return HRT_OK;
}

int hrt_set_field_transform(hrt_handle* h, int32_t identity, const double* field_from_world) {
    if (!h || (!identity && !field_from_world)) return fail(HRT_EINVAL, "null argument");
    if (h->sc.field.kind == HRT_FIELD_NONE) return fail(HRT_EINVAL, "scene has no field");
    DevField& f = h->sc.field;
    if (!identity) {
        if (field_from_world[12] != 0.0 || field_from_world[13] != 0.0 || field_from_world[14] != 0.0 ||
            field_from_world[15] != 1.0)
            return fail(HRT_EINVAL, "field_from_world bottom row must be (0,0,0,1)");
        for (int i = 0; i < 12; ++i) f.inv[i] = field_from_world[i];
    }
    f.identity = identity ? 1 : 0;       // (the occupancy grid lives in the field frame: unchanged)
    ++h->geo_ver;                        // (the shadow entry table's grid covers the field box)
    return HRT_OK;
}

int hrt_l2_peak(hrt_handle* h, double* read_gbs, double* sector_gbs, int64_t* bytes) {
    if (!h || !read_gbs || !sector_gbs) return fail(HRT_EINVAL, "null argument");
    if (h->sc.field.kind != HRT_FIELD_NEURAL) return fail(HRT_EINVAL, "needs a neural field");
    const NeuralField& nf = h->sc.field.nf;
    // (tables larger than 64 MiB - cfg4's 344 MiB - are probed over their first 64 MiB so the
    // buffer stays L2-resident: the probe measures L2, not DRAM)
    const int64_t nbytes = std::min<int64_t>((int64_t)h->tab_entries * h->F * 4, int64_t(64) << 20);
    const int64_t n16 = nbytes / 16;
    const uint4* buf = reinterpret_cast<const uint4*>(nf.table);
    float* sink = nullptr;
    CK(cudaMalloc(&sink, 4));
    const int threads = 512, blocks = h->sm_count * 4;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float ms = 0.f;
    // coalesced streaming reads of the L2-resident table
    const int passes = 8;
    probe::k_l2_read<<<blocks, threads>>>(buf, n16, 1, sink);       // warm: table into L2
    CK(cudaGetLastError());
    CK(cudaEventRecord(e0, 0));
    probe::k_l2_read<<<blocks, threads>>>(buf, n16, passes, sink);
    CK(cudaEventRecord(e1, 0));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *read_gbs = (double)n16 * 16.0 * passes / (ms * 1e-3) / 1e9;
    // random 32-B sector gathers over the same table
    const uint32_t n_sec = (uint32_t)(nbytes / 32);
    const int iters = 64;
    probe::k_sector_gather<<<blocks, threads>>>(buf, n_sec, iters, sink);   // warm
    CK(cudaEventRecord(e0, 0));
    probe::k_sector_gather<<<blocks, threads>>>(buf, n_sec, iters, sink);
    CK(cudaEventRecord(e1, 0));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *sector_gbs = (double)blocks * threads * iters * 8 * 16.0 / (ms * 1e-3) / 1e9;
    if (bytes) *bytes = nbytes;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return HRT_OK;
}

}  // extern "C"


#ifdef HRT_WS_PROFILE
// Dev builds only: read and reset the field-engine cycle counters.
extern "C" int hrt_ws_profile(unsigned long long* out8) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out8, fws::ws_prof, 8 * sizeof(unsigned long long));
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(fws::ws_prof, z, sizeof(z));
    return 0;
}
#endif
