// common.cuh - device-side scene structures and exact-arithmetic helpers.
//
// The whole library is compiled with --fmad=false: every a*b+c that the
// reference (numpy, float64, reference pkg/src/hybridrt) evaluates as two
// roundings stays two roundings here, so ray origins/directions, hit
// distances and BSDF directions reproduce the reference bit-for-bit. The
// few places where the reference itself fuses (the OpenBLAS matmul in
// Camera.primary_rays) use __fma_rn explicitly.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HRT_DEV __device__ __forceinline__

// Checked builds (-DHRT_CHECKS=1, tools/build_checked.sh): device-side bounds
// checks on every queue reservation, batch row, shadow-queue slot and output
// pixel; a violation prints its site and traps (the launch fails with an
// error instead of corrupting memory). compute-sanitizer is not available on
// the GPU pool, so this build is the race / bounds evidence.
#ifndef HRT_CHECKS
#define HRT_CHECKS 0
#endif
#if HRT_CHECKS
#include <cstdio>
#define HRT_ASSERT(cond, what, v, cap)                                                            \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("HRT_CHECKS %s:%d %s: %lld outside [0, %lld)\n", __FILE__, __LINE__, what,     \
                   (long long)(v), (long long)(cap));                                             \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define HRT_ASSERT(cond, what, v, cap) do { } while (0)
#endif

// ----------------------------------------------------------------- vectors
struct d3 { double x, y, z; };
HRT_DEV d3 mk(double x, double y, double z) { return {x, y, z}; }
HRT_DEV d3 add(d3 a, d3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
HRT_DEV d3 sub(d3 a, d3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
HRT_DEV d3 scale(d3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
HRT_DEV d3 neg(d3 a) { return {-a.x, -a.y, -a.z}; }
// numpy np.sum(a*b, axis=1) over a 3-vector: (a0*b0 + a1*b1) + a2*b2
HRT_DEV double dot(d3 a, d3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
// np.linalg.norm(.., axis=1): sqrt((x*x + y*y) + z*z)
HRT_DEV double norm(d3 a) { return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); }
// np.cross: plain mul-sub per component
HRT_DEV d3 cross(d3 a, d3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// --------------------------------------------------------------------- RNG
// Reference hybridrt/rng.py:14-57: h = G; per key h = fmix(h + G ^ (k*B + G));
// u = (h >> 11) * 2^-53 (double). Keys are int64 reinterpreted as uint64.
namespace rng {
constexpr uint64_t G = 0x9E3779B97F4A7C15ull;
constexpr uint64_t A = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t B = 0x94D049BB133111EBull;
enum Purpose { PIXEL_X = 0, PIXEL_Y = 1, BSDF_LOBE = 2, BSDF_U = 3, BSDF_V = 4,
               LIGHT_PICK = 5, LIGHT_U = 6, LIGHT_V = 7, GENERIC = 8 };
HRT_DEV uint64_t fmix(uint64_t h) {
    h ^= h >> 30; h *= A; h ^= h >> 27; h *= B; return h ^ (h >> 31);
}
HRT_DEV uint64_t step(uint64_t h, int64_t k) {
    return fmix((h + G) ^ ((uint64_t)k * B + G));
}
// (seed, pixel, sample, bounce, purpose, lane)
HRT_DEV double uniform(uint64_t seed, int64_t pix, int64_t smp, int64_t bounce, int64_t purpose,
                       int64_t lane) {
    uint64_t h = G;
    h = step(h, (int64_t)seed); h = step(h, pix); h = step(h, smp);
    h = step(h, bounce); h = step(h, purpose); h = step(h, lane);
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}
// The chain state after (seed, pix, smp, bounce): every draw of one path
// segment shares it (shadow rays of a march: 3 draws per sample).
HRT_DEV uint64_t prefix(uint64_t seed, int64_t pix, int64_t smp, int64_t bounce) {
    uint64_t h = G;
    h = step(h, (int64_t)seed); h = step(h, pix); h = step(h, smp);
    return step(h, bounce);
}
HRT_DEV double uniform_from(uint64_t h4, int64_t purpose, int64_t lane) {
    const uint64_t h = step(step(h4, purpose), lane);
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}
}  // namespace rng

// ------------------------------------------------------------------ scene
struct BvhNode {            // 56 B, float64 bounds (conservatively padded)
    double lo[3];
    double hi[3];
    int32_t first;          // leaf: first triangle (leaf order); inner: left child (right = left+1)
    int32_t count;          // > 0 leaf
};

// Traversal node: both children's boxes inline in float32, rounded outward
// and padded (see hrt.cu wbox), so one 64-byte load decides both children.
// ref >= 0: inner node index; ref < 0: leaf ~((first << 3) | count).
struct __align__(16) WNode {
    float4 a;   // lo0.x lo0.y lo0.z hi0.x
    float4 b;   // hi0.y hi0.z lo1.x lo1.y
    float4 c;   // lo1.z hi1.x hi1.y hi1.z
    int4 r;     // ref0, ref1, -, -
};

// 4-wide traversal node (the binary WNode tree collapsed): 4 child boxes as
// SoA float4s + refs (same ref encoding; empty slot: ref -1, far point box).
struct __align__(16) QNode {
    float4 lox, loy, loz, hix, hiy, hiz;
    int4 ref;
    int4 pad;
};

struct DevBvh {
    const QNode* qnodes;    // 4-wide float32-culling tree (traversal)
    unsigned long long qtex;   // float4 texture over qnodes (8 texels per node), 0 = none
    const WNode* wnodes;    // binary float32 tree (source of the 4-wide one)
    const BvhNode* nodes;
    const double* tri;      // leaf-ordered: v0, e1, e2 (9 doubles)
    const int32_t* tri_id;  // leaf order -> global face id
    int32_t n_faces;
};

struct DevMaterials {
    const int32_t* kind;    // 0 lambertian, 1 mirror, 2 dielectric
    const double* rgb;      // albedo / reflectance / tint
    const double* ior;
    const double* r0;       // Schlick R0 per material (host: ((ior-1)/(ior+1))**2)
};

struct DevEmitters {
    int32_t n;
    const double* tris;     // n x 9
    const double* cdf;
    const double* r_src;
};

struct DenseGrid {
    int32_t res[3];
    double scale[3];
    const double* sigma;    // C order, z fastest
    const double* rad;      // (.., 3)
    int32_t sigma_const, rad_const;
    double sigma0, rad0[3];
};

struct NeuralLevel {
    float scale[3];
    int32_t n;              // N_l
    uint32_t r;             // N_l + 1 (dense stride)
    int32_t dense;
    int64_t offset;         // entry offset of the level
};

constexpr int kMaxLevels = 16;

struct NeuralField {
    float lo32[3];
    int32_t n_levels, n_features, enc_dim, act;
    uint32_t tmask;
    NeuralLevel lv[kMaxLevels];
    const float* table;
    unsigned long long tex;  // texture object over `table` (F-wide texels), fine-level gathers
    int32_t tex_from;        // levels >= tex_from gather through the TEX pipe
    const uint8_t* wpack;   // UMMA B-operand images of the 5 layers, back to back
    int32_t occ_res;
    float occ_scale[3];
    double occ_cell[3];
    const uint32_t* occ;
};

enum FieldKind { FIELD_NONE = 0, FIELD_DENSE = 1, FIELD_NEURAL = 2 };

struct DevField {
    int32_t kind;
    int32_t identity;
    double lo[3], hi[3];
    double inv[12];         // field_from_world rows 0..2 (rotation | translation)
    DenseGrid dense;
    NeuralField nf;
};

struct DevScene {
    DevBvh bvh;
    DevBvh blockers;
    const double* normal;   // global face order
    const double* emission;
    const int32_t* mesh_of;
    DevMaterials mat;
    DevEmitters em;
    DevField field;
    int32_t n_bounces;
    double threshold, march_step, spawn_eps, early_t;
    int32_t sample_cap;
    // Shadow entry table (bvh::k_shadow_entry, hrt.cu ensure_shadow_entry):
    // for every cell of a g^3 world grid over the field box x emitter x
    // light patch (p x p cells of the (sqrt(u1), u2) sample square), the
    // blocker-tree node under which every triangle that a shadow ray from
    // the cell to the patch can hit lies (-2: none can be hit). Null: off.
    const int32_t* shent;
    int32_t shent_g, shent_p;
    double shent_lo[3], shent_inv[3];
};

// SoA per-path state for one wavefront chunk.
struct PathState {
    double *ox, *oy, *oz, *dx, *dy, *dz;      // current ray
    double *Lr, *Lg, *Lb;                     // radiance
    double *Tr, *Tg, *Tb;                     // channel throughput (T_spec)
    double *Tm;                               // scalar medium throughput
    int32_t* neval;                           // NeRF samples evaluated on the path
    double* t_hit;
    int32_t* face;
    int32_t* pix;                             // pixel id of the path
    int32_t* smp;                             // sample index of the path
    int32_t* queue[2];                        // alive path ids, ping-pong
    int32_t* counters;                        // [0],[1] queue sizes; [2] fetch cursor; [3..] per-round
    unsigned long long* stats;                // whole-call totals (S_*), 64-bit: a 4K x 64 spp
                                              // frame evaluates ~1e11 NeRF samples
};

// S_SHADOW: shadow rays traced (k_shadow casts one per batch row that needs
// it, including rows a later early-out / cap discards); S_SHADOW_USED: the
// ones whose mask was composited (the reference's count, field.py:246-251).
enum Stat { S_SAMPLES = 0, S_SHADOW = 1, S_SEGMENTS = 2, S_EVALS = 3, S_ROWS = 4, S_SHADOW_USED = 8,
            S_COUNT = 10 };

HRT_DEV void stat_add(unsigned long long* stats, int which, long long v) {
    atomicAdd(stats + which, (unsigned long long)v);
}

enum Counter { C_Q0 = 0, C_Q1 = 1, C_FETCH = 2,
               C_NONFINITE = 6, C_TRACE = 7, C_MQ0 = 8, C_MQ1 = 9, C_NS = 10,
               // device-driven march rounds (k_round_begin): current march queue,
               // first-round flag, samples per path, row stride of this and the
               // previous batch
               C_CUR = 12, C_FIRST = 13, C_S = 14, C_STRIDE = 15, C_PSTRIDE = 16,
               // shadow-ray queue of a round: length, fetch cursor of the tracer
               C_SHQ = 17, C_SHF = 18,
               // k_step in tail mode (G lanes per path) this round
               C_TAIL = 19,
               // march-round ordinal of this render call (k_round_begin; hrt_round_rows)
               C_RIDX = 20,
               // k_paths_bounce: lengths of its two ping-pong path queues
               C_PB0 = 21, C_PB1 = 22,
               C_COUNT = 16 };

HRT_DEV d3 field_point(const DevField& f, d3 p) {
    if (f.identity) return p;
    const double* m = f.inv;
    return {__fma_rn(p.z, m[2], __fma_rn(p.y, m[1], p.x * m[0])) + m[3],
            __fma_rn(p.z, m[6], __fma_rn(p.y, m[5], p.x * m[4])) + m[7],
            __fma_rn(p.z, m[10], __fma_rn(p.y, m[9], p.x * m[8])) + m[11]};
}
HRT_DEV d3 field_dir(const DevField& f, d3 d) {
    if (f.identity) return d;
    const double* m = f.inv;
    return {__fma_rn(d.z, m[2], __fma_rn(d.y, m[1], d.x * m[0])),
            __fma_rn(d.z, m[6], __fma_rn(d.y, m[5], d.x * m[4])),
            __fma_rn(d.z, m[10], __fma_rn(d.y, m[9], d.x * m[8]))};
}

// Reference field.py:88-101 (_ray_slab) for one ray: entry/exit t.
HRT_DEV void slab(const double* lo, const double* hi, d3 o, d3 d, double& t0, double& t1) {
    const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
    t0 = -INFINITY; t1 = INFINITY;
    for (int a = 0; a < 3; ++a) {
        double near, far;
        if (dd[a] == 0.0) {
            bool out = (oo[a] < lo[a]) || (oo[a] > hi[a]);
            near = out ? INFINITY : -INFINITY;
            far = out ? -INFINITY : INFINITY;
        } else {
            double inv = 1.0 / dd[a];
            double ta = (lo[a] - oo[a]) * inv, tb = (hi[a] - oo[a]) * inv;
            near = fmin(ta, tb); far = fmax(ta, tb);
        }
        t0 = fmax(t0, near); t1 = fmin(t1, far);
    }
}

HRT_DEV bool inside_box(const double* lo, const double* hi, d3 p) {
    return p.x >= lo[0] && p.x <= hi[0] && p.y >= lo[1] && p.y <= hi[1] && p.z >= lo[2] &&
           p.z <= hi[2];
}
