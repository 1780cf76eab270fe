// kernels.cuh - the wavefront render pipeline (one chunk of camera paths).
// Neural field, hybrid mode (the continuous march, default):
//   k_raygen -> k_paths (every bounce's ray + nearest hit) -> k_seg ->
//   rounds of { k_round_begin -> k_step (composite, shade/advance, generate)
//               -> fws::k_field_ws -> [k_shadow -> k_shadow_trace] } -> k_accumulate
// Other fields / modes, and the reference's bounce-by-bounce schedule:
//   k_raygen -> per bounce { k_intersect -> march (dense: k_march_dense) -> k_shade }
//   -> k_accumulate
// Path state is SoA in HBM; the alive sets are ping-pong index queues whose
// lengths live on the device, so rounds launch without host syncs (the host
// checks for completion every few rounds).
#pragma once
#include <cooperative_groups.h>
#include "bvh.cuh"
#include "common.cuh"
#include "field_neural.cuh"
#include "field_ws.cuh"
#include "path.cuh"

namespace cg = cooperative_groups;

namespace kern {

struct Args {
    DevScene sc;
    PathState ps;
    path::Camera cam;
    const int32_t* pixels;   // pixel id per slot (nullptr: slot + pixel_base)
    int64_t pixel_base;
    int64_t n_slots;         // pixels in this chunk
    int32_t spp, strat;
    uint64_t seed;
    int32_t bounce;          // 1-based
    int32_t cur;             // current queue (0/1)
    int32_t volume;          // degenerate tracer B: no surfaces, t_hit = inf
    double* out;             // (n_slots, 3) device output
    int64_t out_offset;      // slot offset in `out`
    int32_t tiled;           // full frame: slots walk 16x16 pixel tiles, out is raster
    int32_t out_by_pixel;    // out is a raster frame indexed by global pixel id (may be a peer GPU's)
    int32_t* trace;          // optional (path, bounce, k, cell) records
    int64_t trace_cap;
    int32_t mixed;           // continuous wavefront march: bounces advance inside k_step
};

// One of a two-entry pointer array in a kernel parameter. A plain
// arr[runtime index] makes the compiler copy the whole parameter struct to
// local memory (ncu: STL of every field at kernel entry).
template <class T>
HRT_DEV T* pick(T* const (&arr)[2], int32_t i) { return i ? arr[1] : arr[0]; }

// Warp-aggregated reservation of `n` slots on a device counter.
HRT_DEV int32_t reserve(int32_t* ctr) {
    cg::coalesced_group g = cg::coalesced_threads();
    int32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, (int32_t)g.size());
    base = g.shfl(base, 0);
    return base + (int32_t)g.thread_rank();
}

// Full-frame slot order: 16x16 pixel tiles in raster tile order, raster
// inside a tile (edge tiles partial). Consecutive paths are then a compact
// 2-D pixel block, so a 128-row sample tile of the field engine gathers a
// 16x8 footprint instead of a 128x1 strip (L1 reuse of the mid hash levels).
// Paths are keyed by pixel, so the order never changes a result.
constexpr int kTile = 16;
HRT_DEV int64_t tiled_pixel(int64_t slot, int32_t W, int32_t H) {
    const int64_t band = (int64_t)W * kTile;
    const int64_t ty = slot / band;
    const int64_t rem = slot - ty * band;
    const int64_t ht = min((int64_t)kTile, (int64_t)H - ty * kTile);
    const int64_t tx = rem / (kTile * ht);
    const int64_t r2 = rem - tx * kTile * ht;
    const int64_t wt = min((int64_t)kTile, (int64_t)W - tx * kTile);
    return (ty * kTile + r2 / wt) * W + tx * kTile + r2 % wt;
}

HRT_DEV int64_t slot_pixel(const Args& a, int64_t slot) {
    if (a.pixels) return a.pixels[slot];
    const int64_t s = a.pixel_base + slot;
    return a.tiled ? tiled_pixel(s, a.cam.width, a.cam.height) : s;
}

__global__ void k_raygen(Args a) {
    const int64_t n = a.n_slots * a.spp;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = p / a.spp, smp = p % a.spp;
        const int64_t pix = slot_pixel(a, slot);
        d3 o, d;
        path::primary_ray(a.cam, pix, smp, a.seed, a.strat, o, d);
        PathState& s = a.ps;
        s.ox[p] = o.x; s.oy[p] = o.y; s.oz[p] = o.z;
        s.dx[p] = d.x; s.dy[p] = d.y; s.dz[p] = d.z;
        s.Lr[p] = s.Lg[p] = s.Lb[p] = 0.0;
        s.Tr[p] = s.Tg[p] = s.Tb[p] = 1.0;
        s.Tm[p] = 1.0;
        s.neval[p] = 0;
        s.pix[p] = (int32_t)pix;
        s.smp[p] = (int32_t)smp;
        s.t_hit[p] = INFINITY;
        s.face[p] = -1;
        s.queue[0][p] = (int32_t)p;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ps.counters[C_Q0] = (int32_t)n;
        a.ps.counters[C_Q1] = 0;
    }
}

// trace_path (render.py:302-312): caller-supplied rays instead of camera rays.
__global__ void k_load_rays(Args a, const double* o, const double* d, const int64_t* pix,
                            const int64_t* smp) {
    const int64_t n = a.n_slots;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        PathState& s = a.ps;
        s.ox[p] = o[3 * p]; s.oy[p] = o[3 * p + 1]; s.oz[p] = o[3 * p + 2];
        s.dx[p] = d[3 * p]; s.dy[p] = d[3 * p + 1]; s.dz[p] = d[3 * p + 2];
        s.Lr[p] = s.Lg[p] = s.Lb[p] = 0.0;
        s.Tr[p] = s.Tg[p] = s.Tb[p] = 1.0;
        s.Tm[p] = 1.0;
        s.neval[p] = 0;
        s.pix[p] = (int32_t)pix[p];
        s.smp[p] = (int32_t)smp[p];
        s.t_hit[p] = INFINITY;
        s.face[p] = -1;
        s.queue[0][p] = (int32_t)p;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ps.counters[C_Q0] = (int32_t)n;
        a.ps.counters[C_Q1] = 0;
    }
}

// K2: nearest hit of every alive path, t in (0, inf] (render.py:217).
__global__ void k_intersect(Args a) {
    const int32_t n = a.ps.counters[a.cur];
    const int32_t* q = pick(a.ps.queue, a.cur);
    PathState& s = a.ps;
    if (blockIdx.x == 0 && threadIdx.x == 0) stat_add(s.stats, S_SEGMENTS, n);
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        double t = INFINITY;
        int32_t f = -1;
        if (!a.volume)
            f = bvh::nearest(a.sc.bvh, mk(s.ox[p], s.oy[p], s.oz[p]), mk(s.dx[p], s.dy[p], s.dz[p]),
                             0.0, INFINITY, t);
        s.t_hit[p] = t;
        s.face[p] = f;
    }
}

// --------------------------------------------------------------- march
// Segment of path p: [max(t0, 0), min(t1, t_hit)] against the field box
// (render.py:142-148), midpoint count n = ceil(seg/dt) (field.py:218-220).
struct Segment {
    double s0, delta;
    int32_t n;
};

HRT_DEV bool segment(const DevScene& sc, d3 o, d3 d, double t_end, Segment& g) {
    const DevField& f = sc.field;
    double t0, t1;
    slab(f.lo, f.hi, field_point(f, o), field_dir(f, d), t0, t1);
    const double s0 = fmax(t0, 0.0), s1 = fmin(t1, t_end);
    if (!(s1 > s0)) return false;
    const double seg = fmax(s1 - s0, 0.0);
    double n = ceil(seg / sc.march_step);
    if (seg > 0.0) n = fmax(n, 1.0); else n = 0.0;
    g.s0 = s0;
    g.n = (int32_t)n;
    g.delta = seg / n;
    return g.n > 0;
}

HRT_DEV d3 sample_point(d3 o, d3 d, const Segment& g, int32_t k) {
    const double t = g.s0 + ((double)k + 0.5) * g.delta;
    return {o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
}

struct Acc {
    double L[3], Ts[3], T;
    int32_t neval;
};

HRT_DEV void load_acc(const PathState& s, int32_t p, Acc& c) {
    c.L[0] = s.Lr[p]; c.L[1] = s.Lg[p]; c.L[2] = s.Lb[p];
    c.Ts[0] = s.Tr[p]; c.Ts[1] = s.Tg[p]; c.Ts[2] = s.Tb[p];
    c.T = s.Tm[p];
    c.neval = s.neval[p];
}
HRT_DEV void store_acc(const PathState& s, int32_t p, const Acc& c) {
    s.Lr[p] = c.L[0]; s.Lg[p] = c.L[1]; s.Lb[p] = c.L[2];
    s.Tr[p] = c.Ts[0]; s.Tg[p] = c.Ts[1]; s.Tb[p] = c.Ts[2];
    s.Tm[p] = c.T;
    s.neval[p] = c.neval;
}

// A shadow ray is cast for a midpoint only where it can contribute
// (field.py:246-251: opacity > 0 and max(rgb) > 0).
HRT_DEV bool needs_shadow(const DevScene& sc, double al, const double rgb[3]) {
    return sc.em.n > 0 && al > 0.0 && fmax(fmax(rgb[0], rgb[1]), rgb[2]) > 0.0;
}

// field.py:244-255 for one evaluated midpoint sample with its mask m.
HRT_DEV void composite_m(Acc& c, double al, const double rgb[3], double m) {
    const double am = al * m;
    for (int ch = 0; ch < 3; ++ch) c.L[ch] = c.L[ch] + (c.Ts[ch] * am) * rgb[ch];
    const double keep = 1.0 - al;
    for (int ch = 0; ch < 3; ++ch) c.Ts[ch] = c.Ts[ch] * keep;
    c.T = c.T * keep;
}

// Same with the shadow ray traced inline (dense-grid plugin path).
HRT_DEV void composite(const Args& a, Acc& c, double sigma, const double rgb[3], double delta,
                       d3 p, int32_t pix, int32_t smp, int32_t k) {
    const double al = 1.0 - exp(-sigma * delta);
    double m = 1.0;
    if (needs_shadow(a.sc, al, rgb)) {
        m = path::shadow_mask(a.sc, p, a.seed, pix, smp, a.bounce, k);
        stat_add(a.ps.stats, S_SHADOW, 1);
        stat_add(a.ps.stats, S_SHADOW_USED, 1);
    }
    const double am = al * m;
    for (int ch = 0; ch < 3; ++ch) c.L[ch] = c.L[ch] + (c.Ts[ch] * am) * rgb[ch];
    const double keep = 1.0 - al;
    for (int ch = 0; ch < 3; ++ch) c.Ts[ch] = c.Ts[ch] * keep;
    c.T = c.T * keep;
}

HRT_DEV bool halted(const DevScene& sc, const Acc& c) {
    if (sc.early_t > 0.0 && fmax(fmax(c.Ts[0], c.Ts[1]), c.Ts[2]) < sc.early_t) return true;
    if (sc.sample_cap > 0 && c.neval >= sc.sample_cap) return true;
    return false;
}

// Reference field plugin (dense RadianceGrid): one thread marches one path
// through every midpoint of its segment, as march_arrays does.
__global__ void k_march_dense(Args a) {
    const int32_t n = a.ps.counters[a.cur];
    const int32_t* q = pick(a.ps.queue, a.cur);
    const PathState& s = a.ps;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        const d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
        Segment g;
        if (!segment(a.sc, o, d, s.t_hit[p], g)) continue;
        Acc c;
        load_acc(s, p, c);
        const int32_t pix = s.pix[p], smp = s.smp[p];
        int32_t evals = 0;
        for (int32_t k = 0; k < g.n; ++k) {
            if (halted(a.sc, c)) break;
            const d3 x = sample_point(o, d, g, k);
            double rgb[3];
            const double sigma = path::dense_sample(a.sc.field, x, rgb);
            c.neval += 1;
            ++evals;
            composite(a, c, sigma, rgb, g.delta, x, pix, smp, k);
        }
        store_acc(s, p, c);
        stat_add(a.ps.stats, S_SAMPLES, evals);
    }
}

// Occupancy DDA step: from an empty (or outside) sample k, the first index
// that might leave the current cell. The cell box is shrunk by 1e-4 of a cell
// so float32 cell assignment of later samples cannot disagree; one sample of
// slack covers rounding of t. Every candidate is re-tested by position, so
// the evaluated set equals the oracle's per-sample test exactly.
HRT_DEV int32_t dda_next(const NeuralField& nf, const DevField& f, d3 of, d3 df, const Segment& g,
                         int32_t k, const int32_t cell[3]) {
    double lo[3], hi[3];
    for (int ax = 0; ax < 3; ++ax) {
        const double eps = 1e-4 * nf.occ_cell[ax];
        lo[ax] = f.lo[ax] + (double)cell[ax] * nf.occ_cell[ax] + eps;
        hi[ax] = f.lo[ax] + (double)(cell[ax] + 1) * nf.occ_cell[ax] - eps;
    }
    double t0, t1;
    slab(lo, hi, of, df, t0, t1);
    if (!(t1 > t0)) return k + 1;
    const double kk = ceil((t1 - g.s0) / g.delta - 0.5) - 1.0;
    if (!(kk > (double)(k + 1))) return k + 1;
    return kk >= (double)g.n ? g.n : (int32_t)kk;
}

// ------------------------------------------------------ NeRF march rounds
// The paper's NeRF march as a three-kernel round (SURVEY K4/K7 around the
// field engine fws::k_field_ws):
//   k_seg   once per bounce: segment [max(t0,0), min(t1,t_hit)], n, delta,
//           field-frame fp32 direction; paths with a segment enter march queue 0
//   k_gen   per round: each marching path walks (occupancy DDA) to its next
//           <= kRoundSamples evaluable midpoints and appends them to the batch
//   (k_field_ws evaluates the batch: encode + tcgen05 MLP)
//   k_comp  per round: each path composites its samples in k order (fp64),
//           with shadows, early-out and sample cap; unfinished paths go to
//           the other march queue
// The evaluated sample set and the compositing order equal the oracle's
// per-sample march (oracle/tracer.py march), so parity is unchanged.
#ifndef HRT_ROUND_SAMPLES
#define HRT_ROUND_SAMPLES 24
#endif
// max midpoints per path per round (cfg3 frame 16 / 20 / 24 / 28 / 32 / 40: 197.1 / 195.8 /
// 196.5 / 198.3 / 199.9 / 201.2 ms; cfg1 14.0 / 13.8 / 13.4 / 13.3 / 13.4 / 13.4 ms; 24 also
// the fastest at every 1-8-GPU rank share of cfg3)
constexpr int kRoundSamples = HRT_ROUND_SAMPLES;
#ifndef HRT_ROUND_SAMPLES_SMALL
#define HRT_ROUND_SAMPLES_SMALL 48
#endif
#ifndef HRT_SMALL_LIVE
#define HRT_SMALL_LIVE 200000
#endif
constexpr int kRoundSamplesSmall = HRT_ROUND_SAMPLES_SMALL;   // ... when fewer than kSmallLive paths march
constexpr int kSmallLive = HRT_SMALL_LIVE;

// Ray geometry of every bounce of a path, traced ahead of the march
// (continuous march): bounce b (1-based) of path p at [(b - 1) * cap + p].
struct PathGeo {
    double *ox, *oy, *oz, *dx, *dy, *dz, *t;    // ray of bounce b (b >= 2) and its nearest-hit t
    int32_t* face;                              // nearest face of bounce b (-1: miss)
    int64_t cap;
};

struct MarchState {         // per path, valid while the path is marching
    double* s0;
    double* delta;
    int32_t* n;
    int32_t* k;             // next candidate midpoint
    int32_t* base;          // batch slice of the current round
    int32_t* cnt;
    float4* dir32;          // field-frame direction (SH input)
    int32_t* mq[2];         // march queues
    fws::SampleIn* in;      // batch
    int32_t* sk;            // midpoint index of each batch sample
    float4* out;            // (sigma, rgb) of each batch sample
    int32_t* shadow;        // per batch sample: 0 visible / 1 + blocked emitter index
    struct QRay* shq;       // shadow rays that reach the blocker tree (k_shadow_trace)
    uint64_t* h4;           // per path: rng::prefix(seed, pix, smp, bounce) of this bounce
    int32_t* bounce;        // per path: its current bounce (continuous wavefront march)
    PathGeo geo;            // per path and bounce: ray + nearest hit (k_paths)
    int64_t rows_cap;       // batch rows allocated (HRT_CHECKS)
    int64_t paths_cap;      // path slots allocated (HRT_CHECKS)
};

#define HRT_CHECK_ROW(m, row) HRT_ASSERT((row) >= 0 && (row) < (m).rows_cap, "batch row", row, (m).rows_cap)
#define HRT_CHECK_SLOT(m, r) HRT_ASSERT((r) >= 0 && (r) < (m).paths_cap, "queue slot", r, (m).paths_cap)

// A queued shadow ray (64 B): origin = the NeRF sample point, float64 as the
// reference; row of the batch sample it decides.
struct __align__(16) QRay {
    double ox, oy, oz, dx, dy, dz, tmax;
    int32_t row, idx;
};

// K8 (render.py:221-244) in two parts. The next ray depends only on the
// geometry (hit, normal, material) and the keyed RNG, never on the march, so
// it can be formed ahead of the march (k_paths); the weight update needs the
// post-march throughput.
//
// spawn_ray: normal flip, BSDF sample (RNG keys (pix, smp, bounce)), spawn
// point + spawn_eps * new direction.
HRT_DEV void spawn_ray(const Args& a, int32_t pix, int32_t smp, int32_t bounce, d3 o, d3 d, double t,
                       int32_t f, d3& o2, d3& d2) {
    const DevScene& sc = a.sc;
    const d3 point = {o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
    const d3 n_raw = mk(sc.normal[3 * f], sc.normal[3 * f + 1], sc.normal[3 * f + 2]);
    const bool facing = dot(n_raw, d) < 0.0;
    const d3 nrm = facing ? n_raw : neg(n_raw);
    const int32_t mi = sc.mesh_of[f];
    const int32_t kind = sc.mat.kind[mi];
    const d3 wo = neg(d);
    d3 nd;
    if (kind == 0) {
        const double u1 = rng::uniform(a.seed, pix, smp, bounce, rng::BSDF_U, 0);
        const double u2 = rng::uniform(a.seed, pix, smp, bounce, rng::BSDF_V, 0);
        nd = path::cosine_sample(nrm, u1, u2);
    } else if (kind == 1) {
        nd = path::reflect(wo, nrm);
    } else {
        const double u = rng::uniform(a.seed, pix, smp, bounce, rng::BSDF_LOBE, 0);
        nd = path::dielectric_sample(wo, nrm, facing, sc.mat.ior[mi], sc.mat.r0[mi], u);
    }
    o2 = {point.x + sc.spawn_eps * nd.x, point.y + sc.spawn_eps * nd.y, point.z + sc.spawn_eps * nd.z};
    d2 = nd;
}

// shade_weight: emission of a front-facing hit with the post-march T_spec,
// T_spec *= albedo / reflectance / tint. True if the path goes on
// (max(T_spec) >= threshold).
HRT_DEV bool shade_weight(const DevScene& sc, int32_t f, d3 d, Acc& c) {
    const d3 n_raw = mk(sc.normal[3 * f], sc.normal[3 * f + 1], sc.normal[3 * f + 2]);
    if (dot(n_raw, d) < 0.0) {
        c.L[0] = c.L[0] + c.Ts[0] * sc.emission[3 * f];
        c.L[1] = c.L[1] + c.Ts[1] * sc.emission[3 * f + 1];
        c.L[2] = c.L[2] + c.Ts[2] * sc.emission[3 * f + 2];
    }
    const int32_t mi = sc.mesh_of[f];
    for (int ch = 0; ch < 3; ++ch) c.Ts[ch] = c.Ts[ch] * sc.mat.rgb[3 * mi + ch];
    return fmax(fmax(c.Ts[0], c.Ts[1]), c.Ts[2]) >= sc.threshold;
}

// Both parts in place (the per-bounce k_shade).
HRT_DEV bool shade_one(const Args& a, int32_t p, int32_t bounce, Acc& c) {
    const PathState& s = a.ps;
    const int32_t f = s.face[p];
    if (f < 0) return false;
    const d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
    d3 o2, d2;
    spawn_ray(a, s.pix[p], s.smp[p], bounce, o, d, s.t_hit[p], f, o2, d2);
    const bool go = shade_weight(a.sc, f, d, c);
    s.ox[p] = o2.x; s.oy[p] = o2.y; s.oz[p] = o2.z;
    s.dx[p] = d2.x; s.dy[p] = d2.y; s.dz[p] = d2.z;
    return go;
}

// K2 for all bounces of every path: nearest hit of bounce 1, then while the
// ray hits and bounces remain, the spawned ray of the next bounce and its
// hit. Same arithmetic as intersect -> shade -> intersect (bit-identical
// rays); paths later cut by the throughput threshold just leave unused rays.
#ifndef HRT_PATHS_MINB
#define HRT_PATHS_MINB 4
#endif
// 64 registers (4 blocks of 256 per SM): cfg3 (1.02 M triangles) -18 % vs 90 registers
#ifndef HRT_PATHS_THREADS
#define HRT_PATHS_THREADS 128
#endif
__global__ void __launch_bounds__(HRT_PATHS_THREADS, HRT_PATHS_MINB * 256 / HRT_PATHS_THREADS) k_paths(Args a, PathGeo g) {
    const int32_t n = a.ps.counters[C_Q0];
    const int32_t* q = a.ps.queue[0];
    const PathState& s = a.ps;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
        const int32_t pix = s.pix[p], smp = s.smp[p];
        for (int32_t b = 1; b <= a.sc.n_bounces; ++b) {
            double t = INFINITY;
            const int32_t f = bvh::nearest(a.sc.bvh, o, d, 0.0, INFINITY, t);
            const int64_t at = (int64_t)(b - 1) * g.cap + p;
            g.t[at] = t;
            g.face[at] = f;
            if (b == 1) {
                s.t_hit[p] = t;
                s.face[p] = f;
            }
            if (f < 0 || b == a.sc.n_bounces) break;
            d3 o2, d2;
            spawn_ray(a, pix, smp, b, o, d, t, f, o2, d2);
            o = o2;
            d = d2;
            const int64_t nx = at + g.cap;
            g.ox[nx] = o.x; g.oy[nx] = o.y; g.oz[nx] = o.z;
            g.dx[nx] = d.x; g.dy[nx] = d.y; g.dz[nx] = d.z;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) stat_add(s.stats, S_SEGMENTS, n);   // bounce-1 rays
}

// k_paths bounce by bounce: one launch per bounce b traces the bounce-b rays
// of the paths in qin (bounce 1: every path of queue 0; later: the paths
// whose bounce b-1 ray hit) and compacts the paths that go on into qout, so
// a warp's lanes all carry live rays instead of idling once their own path
// has missed. Same rays, hits and spawn arithmetic as k_paths.
__global__ void __launch_bounds__(HRT_PATHS_THREADS, HRT_PATHS_MINB * 256 / HRT_PATHS_THREADS)
k_paths_bounce(Args a, PathGeo g, int32_t b, const int32_t* __restrict__ qin, const int32_t* nin,
               int32_t* __restrict__ qout, int32_t* nout) {
    const int32_t n = *nin;
    const PathState& s = a.ps;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t p = qin[j];
        const int64_t at = (int64_t)(b - 1) * g.cap + p;
        const d3 o = b == 1 ? mk(s.ox[p], s.oy[p], s.oz[p]) : mk(g.ox[at], g.oy[at], g.oz[at]);
        const d3 d = b == 1 ? mk(s.dx[p], s.dy[p], s.dz[p]) : mk(g.dx[at], g.dy[at], g.dz[at]);
        double t = INFINITY;
        const int32_t f = bvh::nearest(a.sc.bvh, o, d, 0.0, INFINITY, t);
        g.t[at] = t;
        g.face[at] = f;
        if (b == 1) {
            s.t_hit[p] = t;
            s.face[p] = f;
        }
        if (f < 0 || b == a.sc.n_bounces) continue;
        d3 o2, d2;
        spawn_ray(a, s.pix[p], s.smp[p], b, o, d, t, f, o2, d2);
        const int64_t nx = at + g.cap;
        g.ox[nx] = o2.x; g.oy[nx] = o2.y; g.oz[nx] = o2.z;
        g.dx[nx] = d2.x; g.dy[nx] = d2.y; g.dz[nx] = d2.z;
        qout[reserve(nout)] = p;
    }
    if (b == 1 && blockIdx.x == 0 && threadIdx.x == 0) stat_add(s.stats, S_SEGMENTS, n);   // bounce-1 rays
}

// k_paths with 4 lanes per path (bvh::closest_q_coop), for chunks of few
// paths where the longest per-path chain of traversals bounds the launch.
__global__ void __launch_bounds__(256) k_paths_coop(Args a, PathGeo g) {
    const int32_t n = a.ps.counters[C_Q0];
    const int32_t* q = a.ps.queue[0];
    const PathState& s = a.ps;
    const uint32_t lane = threadIdx.x & 31u, gl = lane & 3u, gbase = lane - gl;
    const uint32_t gmask = 0xFu << gbase;
    const int32_t groups = (int32_t)(gridDim.x * blockDim.x / 4);
    for (int32_t j = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) / 4); j < n; j += groups) {
        const int32_t p = q[j];
        d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
        const int32_t pix = s.pix[p], smp = s.smp[p];
        for (int32_t b = 1; b <= a.sc.n_bounces; ++b) {
            double t = INFINITY;
            const int32_t f = bvh::closest_q_coop(a.sc.bvh, o, d, 0.0, INFINITY, t, gmask, gbase, gl);
            const int64_t at = (int64_t)(b - 1) * g.cap + p;
            if (gl == 0) {
                g.t[at] = t;
                g.face[at] = f;
                if (b == 1) {
                    s.t_hit[p] = t;
                    s.face[p] = f;
                }
            }
            if (f < 0 || b == a.sc.n_bounces) break;
            d3 o2, d2;
            spawn_ray(a, pix, smp, b, o, d, t, f, o2, d2);
            o = o2;
            d = d2;
            if (gl == 0) {
                const int64_t nx = at + g.cap;
                g.ox[nx] = o.x; g.oy[nx] = o.y; g.oz[nx] = o.z;
                g.dx[nx] = d.x; g.dy[nx] = d.y; g.dz[nx] = d.z;
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) stat_add(s.stats, S_SEGMENTS, n);   // bounce-1 rays
}

// Segment set-up of path p for the march of bounce `bounce`; false (n = 0)
// when the ray has no segment inside the field box before its hit.
HRT_DEV bool seg_one(const Args& a, const MarchState& m, int32_t p, int32_t bounce) {
    const PathState& s = a.ps;
    const d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
    Segment g;
    if (!segment(a.sc, o, d, s.t_hit[p], g)) {
        m.n[p] = 0;
        m.k[p] = 0;
        return false;
    }
    m.s0[p] = g.s0;
    m.delta[p] = g.delta;
    m.n[p] = g.n;
    m.k[p] = 0;
    const d3 df = field_dir(a.sc.field, d);
    m.dir32[p] = make_float4((float)df.x, (float)df.y, (float)df.z, 0.f);
    if (m.shq) m.h4[p] = rng::prefix(a.seed, s.pix[p], s.smp[p], bounce);
    return true;
}

// Paths with a segment enter march queue 0; with a.mixed every path does
// (k_step then shades and advances those without one).
__global__ void k_seg(Args a, MarchState m) {
    const int32_t n = a.ps.counters[a.cur];
    const int32_t* q = pick(a.ps.queue, a.cur);
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        const bool has = seg_one(a, m, p, a.bounce);
        if (a.mixed) m.bounce[p] = a.bounce;
        if (has || a.mixed) m.mq[0][reserve(&a.ps.counters[C_MQ0])] = p;
    }
}

// Generate up to S evaluable midpoints of path p (queue rank j of nq) into
// the sample-major batch: the i-th sample goes to row i * nq + j, so a warp's
// lanes are neighbouring paths (adjacent pixels) at the same step -> coherent
// table gathers. Unused rows of the path become holes (path = -1) that the
// field engine skips. Returns the count.
// Batch rows are written once and read by the next kernel: streaming
// stores (evict-first), so they do not push the hash table out of L2.
#ifndef HRT_STREAM_ROWS
#define HRT_STREAM_ROWS 1
#endif
HRT_DEV void st_row(fws::SampleIn* p, const fws::SampleIn& r) {
    if (HRT_STREAM_ROWS) __stcs(reinterpret_cast<float4*>(p), *reinterpret_cast<const float4*>(&r));
    else *p = r;
}

HRT_DEV int32_t gen_path(const Args& a, const MarchState& m, int32_t p, int32_t j, int32_t nq,
                         int32_t S, const Acc& c) {
    const PathState& s = a.ps;
    const DevField& fld = a.sc.field;
    const NeuralField& nf = fld.nf;
    int32_t budget = S;
    if (a.sc.sample_cap > 0) budget = min(budget, a.sc.sample_cap - c.neval);
    int32_t cnt = 0, k = m.k[p];
    if (!halted(a.sc, c)) {
        const d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
        Segment g{m.s0[p], m.delta[p], m.n[p]};
        const d3 of = field_point(fld, o), df = field_dir(fld, d);
        while (cnt < budget && k < g.n) {
            const d3 xf = field_point(fld, sample_point(o, d, g, k));
            if (!inside_box(fld.lo, fld.hi, xf)) { ++k; continue; }
            int32_t cell3[3];
            const int32_t cell = nerf::occ_cell(nf, xf, cell3);
            if (nerf::occ_test(nf, cell)) {
                const float3 p32 = nerf::to_f32(xf);
                fws::SampleIn r;
                r.x = p32.x; r.y = p32.y; r.z = p32.z; r.path = p;
                HRT_CHECK_ROW(m, (int64_t)cnt * nq + j);
                st_row(&m.in[(int64_t)cnt * nq + j], r);
                if (a.sc.em.n > 0 || a.trace) m.sk[(int64_t)cnt * nq + j] = k;   // read by shadows / trace only
                ++cnt;
                ++k;
            } else {
                k = dda_next(nf, fld, of, df, g, k, cell3);
            }
        }
    }
    for (int32_t i = cnt; i < S; ++i) {
        fws::SampleIn r;
        r.x = r.y = r.z = 0.f;
        r.path = -1;
        HRT_CHECK_ROW(m, (int64_t)i * nq + j);
        st_row(&m.in[(int64_t)i * nq + j], r);
    }
    m.cnt[p] = cnt;
    m.k[p] = k;
    return cnt;
}

// Composite the cnt samples path p left at rows i * nq + j (field.py:244-255
// per sample, in k order, fp64) with their shadow masks, the sample cap and
// the early-out. Returns true if the path halted inside the batch.
#ifndef HRT_COMP_BATCH
#define HRT_COMP_BATCH 4
#endif
constexpr int32_t kCompBatch = HRT_COMP_BATCH;

template <bool kTrace, bool kShadows = true>
HRT_DEV bool comp_path(const Args& a, const MarchState& m, int32_t p, int32_t j, int32_t nq,
                       int32_t cnt, double delta, Acc& c, int32_t& done, int32_t& shd) {
    bool stop = false;
    // halted() per sample from a running max(T_spec): every channel is
    // scaled by the same keep >= 0 and rounding is monotonic, so
    // round(max * keep) is exactly max(round(T_c * keep)) - the same test
    double tmax = fmax(fmax(c.Ts[0], c.Ts[1]), c.Ts[2]);
    const double early_t = a.sc.early_t;
    const int32_t cap = a.sc.sample_cap;
    // rows are read kCompBatch at a time ahead of the (sequential) halt
    // test, so a path waits one memory latency per batch, not per sample
    for (int32_t i0 = 0; i0 < cnt && !stop; i0 += kCompBatch) {
        float4 fb[kCompBatch];
        int32_t cb[kCompBatch];
#pragma unroll
        for (int32_t u = 0; u < kCompBatch; ++u) {
            const int64_t row = (int64_t)(i0 + u) * nq + j;
            const bool in = i0 + u < cnt;
            fb[u] = in ? __ldcs(&m.out[row]) : make_float4(0.f, 0.f, 0.f, 0.f);
            cb[u] = (kShadows && in && a.sc.em.n > 0) ? __ldcs(&m.shadow[row]) : 0;
        }
#pragma unroll
        for (int32_t u = 0; u < kCompBatch; ++u) {
            const int32_t i = i0 + u;
            if (i >= cnt) break;
            if ((early_t > 0.0 && tmax < early_t) || (cap > 0 && c.neval >= cap)) { stop = true; break; }
            const float4 f = fb[u];
            const double rgb[3] = {(double)f.y, (double)f.z, (double)f.w};
            const double al = 1.0 - exp(-(double)f.x * delta);
            const double mask = (!kShadows || cb[u] == 0) ? 1.0 : path::mask_of(a.sc, cb[u]);
            if (kShadows && needs_shadow(a.sc, al, rgb)) ++shd;
            c.neval += 1;
            ++done;
            composite_m(c, al, rgb, mask);
            tmax = tmax * (1.0 - al);
            if (kTrace) {
                const int64_t row = (int64_t)i * nq + j;
                const int32_t k = m.sk[row];
                const fws::SampleIn r = m.in[row];
                int32_t c3[3];
                const int32_t cell = nerf::occ_cell(a.sc.field.nf, mk(r.x, r.y, r.z), c3);
                const int64_t slot = atomicAdd(&a.ps.counters[C_TRACE], 1);
                if (slot < a.trace_cap)
                    reinterpret_cast<int4*>(a.trace)[slot] = make_int4(p, a.bounce, k, cell);
            }
        }
    }
    return stop;
}

HRT_DEV void warp_stat_add(unsigned long long* stats, int which, int32_t v) {
    const int32_t t = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && t) stat_add(stats, which, t);
}

// Unfused round (used with the debug trace): k_gen -> field -> k_comp.
__global__ void k_gen(Args a, MarchState m, int32_t mcur, int32_t S) {
    const int32_t nq = a.ps.counters[C_MQ0 + mcur];
    const int32_t* q = pick(m.mq, mcur);
    const PathState& s = a.ps;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        Acc c;
        c.Ts[0] = s.Tr[p]; c.Ts[1] = s.Tg[p]; c.Ts[2] = s.Tb[p];
        c.neval = s.neval[p];
        const int32_t cnt = gen_path(a, m, p, j, nq, S, c);
        if (cnt) atomicAdd(&a.ps.counters[C_NS], cnt);
    }
}

#ifndef HRT_COMP_MINB
#define HRT_COMP_MINB 1
#endif
template <bool kTrace>
__global__ void __launch_bounds__(256, HRT_COMP_MINB) k_comp(Args a, MarchState m, int32_t mcur) {
    const int32_t nq = a.ps.counters[C_MQ0 + mcur];
    const int32_t* q = pick(m.mq, mcur);
    int32_t* next = pick(m.mq, mcur ^ 1);
    int32_t* next_n = &a.ps.counters[C_MQ0 + (mcur ^ 1)];
    const PathState& s = a.ps;
    int32_t done = 0, shd = 0;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        Acc c;
        load_acc(s, p, c);
        const bool stop = comp_path<kTrace>(a, m, p, j, nq, m.cnt[p], m.delta[p], c, done, shd);
        store_acc(s, p, c);
        if (!stop && !halted(a.sc, c) && m.k[p] < m.n[p]) next[reserve(next_n)] = p;
    }
    if (done) stat_add(a.ps.stats, S_SAMPLES, done);
    if (shd) stat_add(a.ps.stats, S_SHADOW_USED, shd);
    if (blockIdx.x == 0 && threadIdx.x == 0) stat_add(a.ps.stats, S_EVALS, a.ps.counters[C_NS]);
}

// Fused round: every path of queue mcur first composites the samples it left
// in the previous batch (rows i * prev_nq + base[p]; none on the first
// round), then - if it goes on - takes rank r in the other queue and
// generates its next samples at rows i * nq + r. One pass over the path
// state per round instead of two (k_gen + k_comp); a path whose remaining
// candidates are all empty cells keeps a rank with S hole rows.
// Continuous wavefront march (a.mixed): a path whose segment is over is
// shaded at its hit (shade_one), and if it goes on, its next bounce's ray is
// intersected (K2) and its segment set up here, inside the round, so its
// samples join the same batch as the other paths' instead of waiting for a
// per-bounce tail of small rounds. Every path still runs the reference's
// per-path sequence (march b -> shade b -> intersect b+1 -> march b+1 ...)
// with the same arithmetic, so results are bit-identical to the per-bounce
// loop. Returns true when the path has a segment to march.
HRT_DEV bool advance(const Args& a, const MarchState& m, int32_t p, Acc& c, int32_t& segs) {
    const PathState& s = a.ps;
    int32_t b = m.bounce[p];
    while (true) {
        const int32_t f = s.face[p];
        if (f < 0) return false;
        if (!shade_weight(a.sc, f, mk(s.dx[p], s.dy[p], s.dz[p]), c)) return false;
        if (b >= a.sc.n_bounces) return false;
        ++b;
        m.bounce[p] = b;
        // the next bounce's ray and nearest hit, traced ahead by k_paths
        const int64_t at = (int64_t)(b - 1) * m.geo.cap + p;
        s.ox[p] = m.geo.ox[at]; s.oy[p] = m.geo.oy[at]; s.oz[p] = m.geo.oz[at];
        s.dx[p] = m.geo.dx[at]; s.dy[p] = m.geo.dy[at]; s.dz[p] = m.geo.dz[at];
        s.t_hit[p] = m.geo.t[at];
        s.face[p] = m.geo.face[at];
        ++segs;
        if (seg_one(a, m, p, b) && !halted(a.sc, c)) return true;
        // nothing to march on this bounce (no segment, or halted): its hit next
    }
}

// ---- tail rounds: G lanes per path (continuous march, few marching paths).
// A round's k_step is a per-path serial chain; when few paths remain (the
// last rounds, or a GPU's small share) the SMs idle and that chain is the
// round's floor. Here G lanes split its independent parts - lane i loads
// sample i0 + i and forms its opacity (the fp64 exp), tests candidate k + i
// (position, box, occupancy) - and lane 0 alone runs the compositing
// recurrence and the advance, in the same order with the same operations as
// comp_path / gen_path / advance, so results are bit-identical.
#ifndef HRT_TAIL_LANES
#define HRT_TAIL_LANES 8
#endif
#ifndef HRT_TAIL_LIVE
#define HRT_TAIL_LIVE 2048
#endif
constexpr int kTailLanes = HRT_TAIL_LANES;
constexpr int kTailLive = HRT_TAIL_LIVE;      // k_round_begin: tail mode below this many paths

template <int G>
struct Grp {
    uint32_t gl, gbase, gmask;
    HRT_DEV Grp() {
        const uint32_t lane = threadIdx.x & 31u;
        gl = lane % G;
        gbase = lane - gl;
        gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << gbase;
    }
    template <class T>
    HRT_DEV T bcast(T v, uint32_t src) const { return __shfl_sync(gmask, v, (int)(gbase + src)); }
    HRT_DEV uint32_t ballot(bool v) const { return (__ballot_sync(gmask, v) & gmask) >> gbase; }
};

template <int G, bool kShadows>
HRT_DEV bool comp_path_tail(const Args& a, const MarchState& m, int32_t j, int32_t nq, int32_t cnt,
                            double delta, Acc& c, int32_t& done, int32_t& shd, const Grp<G>& g) {
    bool stop = false;
    double tmax = fmax(fmax(c.Ts[0], c.Ts[1]), c.Ts[2]);
    const double early_t = a.sc.early_t;
    const int32_t cap = a.sc.sample_cap;
    for (int32_t i0 = 0; i0 < cnt && !stop; i0 += G) {
        const int32_t i = i0 + (int32_t)g.gl;
        const int64_t row = (int64_t)i * nq + j;
        const bool in = i < cnt;
        const float4 f = in ? __ldcs(&m.out[row]) : make_float4(0.f, 0.f, 0.f, 0.f);
        const int32_t cb = (kShadows && in && a.sc.em.n > 0) ? __ldcs(&m.shadow[row]) : 0;
        const double al = 1.0 - exp(-(double)f.x * delta);
        const double mask = (!kShadows || cb == 0) ? 1.0 : path::mask_of(a.sc, cb);
        const int32_t nu = min(G, cnt - i0);
        for (int32_t u = 0; u < nu; ++u) {
            const double alu = g.bcast(al, (uint32_t)u), mu = g.bcast(mask, (uint32_t)u);
            const double rgb[3] = {(double)g.bcast(f.y, (uint32_t)u), (double)g.bcast(f.z, (uint32_t)u),
                                   (double)g.bcast(f.w, (uint32_t)u)};
            if (g.gl == 0 && !stop) {
                if ((early_t > 0.0 && tmax < early_t) || (cap > 0 && c.neval >= cap)) {
                    stop = true;
                } else {
                    c.neval += 1;
                    ++done;
                    if (kShadows && needs_shadow(a.sc, alu, rgb)) ++shd;
                    composite_m(c, alu, rgb, mu);
                    tmax = tmax * (1.0 - alu);
                }
            }
        }
        stop = g.bcast((int32_t)stop, 0) != 0;
    }
    return stop;
}

template <int G>
HRT_DEV int32_t gen_path_tail(const Args& a, const MarchState& m, int32_t p, int32_t j, int32_t nq,
                              int32_t S, int32_t neval, bool halt, const Grp<G>& g) {
    const PathState& s = a.ps;
    const DevField& fld = a.sc.field;
    const NeuralField& nf = fld.nf;
    int32_t budget = S;
    if (a.sc.sample_cap > 0) budget = min(budget, a.sc.sample_cap - neval);
    int32_t cnt = 0, k = m.k[p];
    const bool write_k = a.sc.em.n > 0;
    if (!halt) {
        const d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
        const Segment sg{m.s0[p], m.delta[p], m.n[p]};
        const d3 of = field_point(fld, o), df = field_dir(fld, d);
        while (cnt < budget && k < sg.n) {
            const int32_t kk = k + (int32_t)g.gl;
            const d3 xf = field_point(fld, sample_point(o, d, sg, kk));
            const bool ins = kk < sg.n && inside_box(fld.lo, fld.hi, xf);
            int32_t cell3[3] = {0, 0, 0};
            bool ev = false;
            if (ins) ev = nerf::occ_test(nf, nerf::occ_cell(nf, xf, cell3));
            const uint32_t bal = g.ballot(ev);
            const int32_t rank = __popc(bal & ((1u << g.gl) - 1u));
            if (ev && cnt + rank < budget) {
                const float3 p32 = nerf::to_f32(xf);
                fws::SampleIn r;
                r.x = p32.x; r.y = p32.y; r.z = p32.z; r.path = p;
                const int64_t row = (int64_t)(cnt + rank) * nq + j;
                HRT_CHECK_ROW(m, row);
                st_row(&m.in[row], r);
                if (write_k) m.sk[row] = kk;
            }
            const int32_t n_ev = __popc(bal);
            if (cnt + n_ev >= budget) {
                // budget filled: resume after the last candidate taken
                uint32_t b = bal;
                for (int32_t t = 1; t < budget - cnt; ++t) b &= b - 1u;
                k += __ffs(b);
                cnt = budget;
                break;
            }
            cnt += n_ev;
            const int32_t last = min(G, sg.n - k) - 1;     // last candidate tested
            int32_t knext = k + last + 1;
            // an empty cell at the last candidate: skip the rest of it (gen_path's DDA)
            const bool last_ins = g.bcast((int32_t)ins, (uint32_t)last) != 0;
            if (last_ins && !((bal >> last) & 1u)) {
                int32_t kj = 0;
                if ((int32_t)g.gl == last) kj = dda_next(nf, fld, of, df, sg, kk, cell3);
                knext = max(knext, g.bcast(kj, (uint32_t)last));
            }
            k = knext;
        }
    }
    for (int32_t i = cnt + (int32_t)g.gl; i < S; i += G) {
        fws::SampleIn r;
        r.x = r.y = r.z = 0.f;
        r.path = -1;
        HRT_CHECK_ROW(m, (int64_t)i * nq + j);
        st_row(&m.in[(int64_t)i * nq + j], r);
    }
    if (g.gl == 0) {
        m.cnt[p] = cnt;
        m.k[p] = k;
    }
    return cnt;
}

// One tail round of k_step<true>, G lanes per queued path.
template <int G>
HRT_DEV void step_tail(const Args& a, const MarchState& m, int32_t first, int32_t S, int32_t prev_nq,
                       int32_t nq, const int32_t* q, int32_t* next, int32_t* next_n, int32_t& done,
                       int32_t& made, int32_t& held, int32_t& segs, int32_t& shd) {
    const PathState& s = a.ps;
    const Grp<G> g;
    const int32_t groups = (int32_t)(gridDim.x * blockDim.x / G);
    for (int32_t j = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) / G); j < nq; j += groups) {
        const int32_t p = q[j];
        Acc c;
        load_acc(s, p, c);
        int32_t go = 1;
        if (!first) {
            const bool stop = a.sc.em.n > 0
                                  ? comp_path_tail<G, true>(a, m, m.base[p], prev_nq, m.cnt[p], m.delta[p], c, done, shd, g)
                                  : comp_path_tail<G, false>(a, m, m.base[p], prev_nq, m.cnt[p], m.delta[p], c, done, shd, g);
            if (g.gl == 0) go = !stop && !halted(a.sc, c) && m.k[p] < m.n[p];
        } else if (g.gl == 0) {
            go = m.k[p] < m.n[p];
        }
        int32_t neval = 0, halt = 0;
        if (g.gl == 0) {
            if (!go) go = advance(a, m, p, c, segs);
            store_acc(s, p, c);
            neval = c.neval;
            halt = halted(a.sc, c);
        }
        __syncwarp(g.gmask);                     // lane 0's path-state writes -> the group
        go = g.bcast(go, 0);
        if (go) {
            neval = g.bcast(neval, 0);
            halt = g.bcast(halt, 0);
            int32_t r = 0;
            if (g.gl == 0) {
                r = reserve(next_n);
                HRT_CHECK_SLOT(m, r);
                next[r] = p;
                m.base[p] = r;
            }
            r = g.bcast(r, 0);
            const int32_t cnt = gen_path_tail<G>(a, m, p, r, nq, S, neval, halt != 0, g);
            if (g.gl == 0) {
                made += cnt;
                ++held;
            }
        }
    }
}

// 64 registers (8 blocks of 128 per SM, ~200 B of spills) beats 80 (6 blocks, 84 B):
// cfg3 composite 23.1 -> 21.4 ms; cfg1 and cfg4 equal
#ifndef HRT_STEP_MINB
#define HRT_STEP_MINB 4
#endif
template <bool kMixed>
#ifndef HRT_STEP_THREADS
#define HRT_STEP_THREADS 128
#endif
__global__ void __launch_bounds__(HRT_STEP_THREADS, HRT_STEP_MINB * 256 / HRT_STEP_THREADS) k_step(Args a, MarchState m) {
    const int32_t* ctr = a.ps.counters;
    const int32_t mcur = ctr[C_CUR], S = ctr[C_S], prev_nq = ctr[C_PSTRIDE], first = ctr[C_FIRST];
    const int32_t nq = ctr[C_MQ0 + mcur];
    const int32_t* q = pick(m.mq, mcur);
    int32_t* next = pick(m.mq, mcur ^ 1);
    int32_t* next_n = &a.ps.counters[C_MQ0 + (mcur ^ 1)];
    const PathState& s = a.ps;
    int32_t done = 0, made = 0, held = 0, segs = 0, shd = 0;
    if (kMixed && kTailLanes > 1 && ctr[C_TAIL]) {
        step_tail<kTailLanes>(a, m, first, S, prev_nq, nq, q, next, next_n, done, made, held, segs, shd);
    } else
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        Acc c;
        load_acc(s, p, c);
        bool go = true;
        if (!first) {
            // (no emitters: the shadow codes are all 0, compile the mask out)
            const bool stop = a.sc.em.n > 0
                                  ? comp_path<false, true>(a, m, p, m.base[p], prev_nq, m.cnt[p], m.delta[p], c, done, shd)
                                  : comp_path<false, false>(a, m, p, m.base[p], prev_nq, m.cnt[p], m.delta[p], c, done, shd);
            go = !stop && !halted(a.sc, c) && m.k[p] < m.n[p];
        } else if (kMixed) {
            go = m.k[p] < m.n[p];
        }
        if (kMixed && !go) go = advance(a, m, p, c, segs);
        if (!first || kMixed) store_acc(s, p, c);
        if (go) {
            // dense next batch: rank r among the paths that go on; rows
            // i * nq + r (the field engine reads them through a RowMap)
            const int32_t r = reserve(next_n);
            HRT_CHECK_SLOT(m, r);
            next[r] = p;
            m.base[p] = r;
            made += gen_path(a, m, p, r, nq, S, c);
            ++held;
        }
    }
    warp_stat_add(a.ps.stats, S_SAMPLES, done);
    if (a.sc.em.n > 0) warp_stat_add(a.ps.stats, S_SHADOW_USED, shd);
    warp_stat_add(a.ps.stats, S_EVALS, made);
    if (kMixed) warp_stat_add(a.ps.stats, S_SEGMENTS, segs);
    // the host stops the rounds when a round's C_NS is 0: samples made, or
    // (continuous march) paths still holding a rank
    const int32_t any = __reduce_add_sync(0xffffffffu, kMixed ? made + held : made);
    if ((threadIdx.x & 31) == 0 && any) atomicAdd(&a.ps.counters[C_NS], any);
}

// Start node of a queued shadow ray from the shadow entry table
// (bvh::k_shadow_entry): -2 = no blocker can be hit, 0 = the root (table off,
// or x outside the table's grid).
HRT_DEV int32_t shadow_start(const DevScene& sc, d3 x, const path::ShadowRay& r) {
    if (!sc.shent) return 0;
    const int32_t g = sc.shent_g, P = sc.shent_p;
    const double f[3] = {(x.x - sc.shent_lo[0]) * sc.shent_inv[0], (x.y - sc.shent_lo[1]) * sc.shent_inv[1],
                         (x.z - sc.shent_lo[2]) * sc.shent_inv[2]};
    int32_t c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!(f[a] >= 0.0 && f[a] < (double)g)) return 0;
        c[a] = (int32_t)f[a];
    }
    const int32_t pu = min((int32_t)(r.su * P), P - 1), pv = min((int32_t)(r.u2 * P), P - 1);
    const int64_t cell = (int64_t)c[0] + (int64_t)g * (c[1] + (int64_t)g * c[2]);
    return __ldg(sc.shent + ((cell * sc.em.n + r.idx) * P + pv) * P + pu);
}

// K3 over the batch: one thread per sample row (sample-major, so a warp
// traces the shadow rays of 32 neighbouring pixels at the same step). Rows
// that cannot contribute (opacity 0 or black) cast no ray, as in the
// reference (field.py:246-251).
#ifndef HRT_SHADOW_MINB
#define HRT_SHADOW_MINB 4
#endif
#ifndef HRT_SHADOW_PATH_MAJOR
#define HRT_SHADOW_PATH_MAJOR 1
#endif
constexpr bool kShadowPathMajor = HRT_SHADOW_PATH_MAJOR;
__global__ void __launch_bounds__(256, HRT_SHADOW_MINB) k_shadow(Args a, MarchState m, fws::RowMap rm, int64_t rows,
                                                             int32_t dev_rows) {
    const PathState& s = a.ps;
    uint32_t S = 0;
    if (dev_rows) {                  // device-driven round: this round's batch shape
        const int32_t* ctr = a.ps.counters;
        fws::set_rows(rm, ctr[C_MQ0 + (ctr[C_CUR] ^ 1)], ctr[C_STRIDE]);
        S = (uint32_t)ctr[C_S];
        rows = (int64_t)rm.width * S;
    }
    int32_t cast = 0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < rows;
         l += (int64_t)gridDim.x * blockDim.x) {
        int64_t li = l;
        if (kShadowPathMajor && S > 0) {
            // path-major walk (a warp takes consecutive samples of one or two
            // paths): the path state loads are shared, and the queue gets the
            // rays of a path's consecutive samples side by side - similar
            // origins in one tracer warp, which keeps its node fetches in L1
            const uint32_t jj = (uint32_t)l / S;
            li = (int64_t)((uint32_t)l - jj * S) * rm.width + jj;
        }
        const int64_t row = fws::phys_row(rm, li);
        // the row's loads are issued together, then the path's (one latency each,
        // not a chain; a hole row's output and k are read but unused)
        const int32_t p = m.in[row].path;
        const float4 f = m.out[row];
        const int32_t k = m.sk[row];
        if (p < 0) continue;
        const double delta = m.delta[p];
        const d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
        const double s0 = m.s0[p];
        const int32_t nseg = m.n[p];
        const double rgb[3] = {(double)f.y, (double)f.z, (double)f.w};
        const double al = 1.0 - exp(-(double)f.x * delta);
        int32_t code = 0;
        if (needs_shadow(a.sc, al, rgb)) {
            const Segment g{s0, delta, nseg};
            const d3 x = sample_point(o, d, g, k);
            if (m.shq) {
                // queue the ray for k_shadow_trace unless it misses the blocker tree's root
                const path::ShadowRay r = path::shadow_ray_h(a.sc, x, m.h4[p], k);
                const int32_t start = shadow_start(a.sc, x, r);
                if (start == -2) {
                    code = 0;                          // no blocker can be hit (entry table)
                } else if (bvh::root_overlap(a.sc.blockers, x, r.dir, a.sc.spawn_eps, r.tmax)) {
                    QRay q;
                    q.ox = x.x; q.oy = x.y; q.oz = x.z;
                    q.dx = r.dir.x; q.dy = r.dir.y; q.dz = r.dir.z;
                    q.tmax = r.tmax;
                    q.row = (int32_t)row;
                    q.idx = a.sc.shent ? (r.idx | (start << 8)) : r.idx;   // (start node, emitter)
                    const int32_t qs = reserve(&a.ps.counters[C_SHQ]);
                    HRT_CHECK_ROW(m, qs);
                    m.shq[qs] = q;
                    code = -1;                         // decided by k_shadow_trace
                }
            } else {
                code = path::shadow_code(a.sc, x, a.seed, s.pix[p], s.smp[p], a.mixed ? m.bounce[p] : a.bounce, k);
            }
            ++cast;
        }
        if (code >= 0) m.shadow[row] = code;
    }
    if (cast) stat_add(a.ps.stats, S_SHADOW, cast);
}

// Any-hit of the queued shadow rays: persistent warps that refill idle lanes
// from the queue (warp-aggregated fetch once a quarter of the warp is idle)
// and advance every lane one BVH node per iteration, so long traversals do
// not hold the rest of the warp idle. Same culling and float64 triangle
// tests as bvh::any_hit_w: the blocked / visible answer is identical.
#ifndef HRT_SHADOW_ORDERED
#define HRT_SHADOW_ORDERED 1
#endif
constexpr bool kShadowOrdered = HRT_SHADOW_ORDERED;
#ifndef HRT_REFILL_LANES
#define HRT_REFILL_LANES 8
#endif
constexpr int kRefillLanes = HRT_REFILL_LANES;    // idle lanes that trigger a warp refill

#ifndef HRT_SHTRACE_MINB
#define HRT_SHTRACE_MINB 4
#endif
__global__ void __launch_bounds__(256, HRT_SHTRACE_MINB) k_shadow_trace(Args a, MarchState m) {
    const int32_t n = a.ps.counters[C_SHQ];
    int32_t* fetch = &a.ps.counters[C_SHF];
    const DevBvh& b = a.sc.blockers;
    const uint32_t lane = threadIdx.x & 31;
    const double t_min = a.sc.spawn_eps;
    int32_t qi = -1;
    bool exhausted = false;
    d3 o{}, d{};
    double tmax = 0.0;
    bvh::Ray32 r32{};
    float t0 = 0.f, t1 = 0.f;
    int32_t stack[bvh::kStackQ];
    int sp = 0;
    int32_t cur = 0, row = 0, idx = 0;
#ifdef HRT_COUNT_STEPS
    long long n_steps = 0, n_mt = 0, n_blocked = 0, n_traced = 0, my_steps = 0;
#endif
    while (true) {
        const bool idle = qi < 0 && !exhausted;
        const uint32_t need = __ballot_sync(0xffffffffu, idle);
        const uint32_t busy = __ballot_sync(0xffffffffu, qi >= 0);
        if (need && (__popc(need) >= kRefillLanes || busy == 0)) {
            const int leader = __ffs(need) - 1;
            int32_t base = 0;
            if ((int)lane == leader) base = atomicAdd(fetch, __popc(need));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (idle) {
                const int32_t my = base + __popc(need & ((1u << lane) - 1u));
                if (my < n) {
                    const QRay q = m.shq[my];
                    o = mk(q.ox, q.oy, q.oz);
                    d = mk(q.dx, q.dy, q.dz);
                    tmax = q.tmax;
                    row = q.row;
                    idx = a.sc.shent ? (q.idx & 255) : q.idx;
                    r32 = bvh::prep32(o, d);
                    t0 = bvh::t_lo32(t_min);
                    t1 = bvh::t_hi32(tmax);
                    sp = 0;
                    cur = a.sc.shent ? (q.idx >> 8) : 0;    // the entry table's start node
                    qi = my;
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(0xffffffffu, exhausted || qi < 0) && __all_sync(0xffffffffu, exhausted)) break;
        if (qi < 0) continue;
        if (HRT_BVH_WIDTH == 4) {
            // one step of bvh::any_hit_q: either one 4-wide node (hit children pushed
            // far to near, the nearest taken next) or one leaf triangle, so a warp's
            // lanes never serialise several triangle tests behind one node test
            bool blocked = false, done = false;
            if (cur < 0) {
                blocked = bvh::leaf_any(b, cur, o, d, t_min, tmax);
                done = blocked;
            } else {
                const QNode qn = bvh::load_q<true>(b, cur);
                float nr[4];
                uint32_t mk4 = bvh::qchildren(qn, r32, t0, t1, nr);
                while (mk4) {
                    int kb = -1;
                    float tb = -INFINITY;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if ((mk4 >> k & 1u) && nr[k] >= tb) { tb = nr[k]; kb = k; }
                    mk4 &= ~(1u << kb);
                    if (sp < bvh::kStackQ) stack[sp++] = bvh::qref(qn, kb);
                }
            }
#ifdef HRT_COUNT_STEPS
            ++n_steps;
            ++my_steps;
#endif
            if (!done) {
                if (sp > 0) cur = stack[--sp];
                else done = true;
            }
            if (done) {
                m.shadow[row] = blocked ? idx + 1 : 0;
                qi = -1;
#ifdef HRT_COUNT_STEPS
                ++n_traced;
                if (blocked) { ++n_blocked; n_mt += my_steps; }
                my_steps = 0;
#endif
            }
            continue;
        }
        // one node of the traversal (bvh::any_hit_w, unrolled into steps)
        const WNode w = bvh::load_w(b.wnodes, cur);
        bool h0, h1;
        float n0, n1;
        bvh::wchildren(w, r32, t0, t1, h0, h1, n0, n1);
        bool blocked = false;
#ifdef HRT_COUNT_STEPS
        ++n_steps;
        n_mt += (h0 && w.r.x < 0) + (h1 && w.r.y < 0);
#endif
        if (h0 && w.r.x < 0) { blocked = bvh::leaf_any(b, w.r.x, o, d, t_min, tmax); h0 = false; }
        if (!blocked && h1 && w.r.y < 0) {
            blocked = bvh::leaf_any(b, w.r.y, o, d, t_min, tmax);
            h1 = false;
        }
        bool done = blocked;
        if (!done) {
            if (h0 && h1) {
                const bool near0 = !kShadowOrdered || n0 <= n1;    // nearer child first
                if (sp < bvh::kStack) stack[sp++] = near0 ? w.r.y : w.r.x;
                cur = near0 ? w.r.x : w.r.y;
            } else if (h0 || h1) {
                cur = h0 ? w.r.x : w.r.y;
            } else if (sp > 0) {
                cur = stack[--sp];
            } else {
                done = true;
            }
        }
        if (done) {
            m.shadow[row] = blocked ? idx + 1 : 0;
            qi = -1;
#ifdef HRT_COUNT_STEPS
            n_blocked += blocked;
#endif
        }
    }
#ifdef HRT_COUNT_STEPS
    stat_add(a.ps.stats, 5, n_steps);
    stat_add(a.ps.stats, 6, n_mt);
    stat_add(a.ps.stats, 7, n_blocked);
    stat_add(a.ps.stats, 9, n_traced);
#endif
}

// Device-driven march round (no host sync): flip to the queue k_step will
// read, fix its samples per path (kRoundSamples, more for small tail rounds,
// capped by the batch buffer) and the batch strides, empty the next queue.
__global__ void k_round_begin(int32_t* c, unsigned long long* stats, int32_t target_rows,
                              int32_t batch_cap, int64_t* round_rows, int32_t log_cap) {
    const int32_t cur = c[C_CUR] ^ 1;
    c[C_CUR] = cur;
    c[C_FIRST] = c[C_FIRST] == 2 ? 1 : 0;       // 2 = set by k_march_begin
    const int32_t live = c[C_MQ0 + cur];
    // fewer, longer rounds when a GPU's share of paths is small (a round's
    // k_step floor is a per-path serial chain, so it is paid per round)
    int32_t S = live >= kSmallLive ? kRoundSamples : kRoundSamplesSmall;
    if (live > 0) {
        S = max(S, min(target_rows / live, 256));
        S = max(1, min(S, batch_cap / live));
    }
    c[C_S] = S;
    if (round_rows) {                            // round ordinal for the engine's per-round row log
        const int32_t ri = c[C_RIDX]++;
        if (ri < log_cap) {
            round_rows[ri] = 0;                  // (empty rounds stay 0: round i = the i-th engine launch)
            round_rows[log_cap + ri] = (int64_t)stats[S_EVALS];   // samples generated before round i
        }
    }
    c[C_TAIL] = live > 0 && live < kTailLive;
    c[C_PSTRIDE] = c[C_STRIDE];
    c[C_STRIDE] = live;
    c[C_MQ0 + (cur ^ 1)] = 0;
    c[C_NS] = 0;
    c[C_SHQ] = 0;
    c[C_SHF] = 0;
    (void)stats;
}

// Before the first round of a bounce (k_seg fills march queue 0).
__global__ void k_march_begin(int32_t* c) {
    c[C_CUR] = 1;                // k_round_begin flips it to 0
    c[C_FIRST] = 2;
    c[C_MQ0] = 0;
    c[C_STRIDE] = 0;
}

// Start of a march round: empty the batch and the next march queue.
__global__ void k_round_reset(int32_t* counters, int32_t next_mq) {
    counters[C_NS] = 0;
    counters[C_SHQ] = 0;
    counters[C_SHF] = 0;
    counters[C_MQ0 + next_mq] = 0;
}

__global__ void k_shade(Args a) {
    const int32_t n = a.ps.counters[a.cur];
    const int32_t* q = pick(a.ps.queue, a.cur);
    int32_t* next = pick(a.ps.queue, a.cur ^ 1);
    int32_t* next_n = &a.ps.counters[a.cur ^ 1];
    const PathState& s = a.ps;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        if (s.face[p] < 0) continue;
        Acc c;
        load_acc(s, p, c);
        const bool go = shade_one(a, p, a.bounce, c);
        store_acc(s, p, c);
        if (go) next[reserve(next_n)] = p;
    }
}

// ---------------------------------------------- emitter-estimation transport
// _trace_transport (emitters.py:73-111): like k_shade, but a front-facing hit
// records (face, T_spec / spp) for its bounce instead of adding the face's
// emission; k_transport_reduce adds the records into A in the reference's
// np.add.at order.
__global__ void k_shade_transport(Args a, int32_t depth, int32_t* rec_face, double* rec_val) {
    const int32_t n = a.ps.counters[a.cur];
    const int32_t* q = pick(a.ps.queue, a.cur);
    int32_t* next = pick(a.ps.queue, a.cur ^ 1);
    int32_t* next_n = &a.ps.counters[a.cur ^ 1];
    const PathState& s = a.ps;
    const DevScene& sc = a.sc;
    const double inv_spp = 1.0 / (double)a.spp;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int32_t p = q[j];
        const int32_t f = s.face[p];
        if (f < 0) continue;
        const double t = s.t_hit[p];
        const d3 o = mk(s.ox[p], s.oy[p], s.oz[p]), d = mk(s.dx[p], s.dy[p], s.dz[p]);
        const d3 point = {o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
        const d3 n_raw = mk(sc.normal[3 * f], sc.normal[3 * f + 1], sc.normal[3 * f + 2]);
        const bool facing = dot(n_raw, d) < 0.0;
        const d3 nrm = facing ? n_raw : neg(n_raw);
        double T[3] = {s.Tr[p], s.Tg[p], s.Tb[p]};
        if (facing) {
            const int64_t r = (int64_t)p * depth + (a.bounce - 1);
            rec_face[r] = f;
            for (int ch = 0; ch < 3; ++ch) rec_val[3 * r + ch] = T[ch] * inv_spp;
        }
        const int32_t mi = sc.mesh_of[f];
        const int32_t kind = sc.mat.kind[mi];
        const d3 wo = neg(d);
        const int32_t pix = s.pix[p], smp = s.smp[p];
        d3 nd;
        if (kind == 0) {
            const double u1 = rng::uniform(a.seed, pix, smp, a.bounce, rng::BSDF_U, 0);
            const double u2 = rng::uniform(a.seed, pix, smp, a.bounce, rng::BSDF_V, 0);
            nd = path::cosine_sample(nrm, u1, u2);
        } else if (kind == 1) {
            nd = path::reflect(wo, nrm);
        } else {
            const double u = rng::uniform(a.seed, pix, smp, a.bounce, rng::BSDF_LOBE, 0);
            nd = path::dielectric_sample(wo, nrm, facing, sc.mat.ior[mi], sc.mat.r0[mi], u);
        }
        for (int ch = 0; ch < 3; ++ch) T[ch] = T[ch] * sc.mat.rgb[3 * mi + ch];
        s.Tr[p] = T[0]; s.Tg[p] = T[1]; s.Tb[p] = T[2];
        s.ox[p] = point.x + sc.spawn_eps * nd.x;
        s.oy[p] = point.y + sc.spawn_eps * nd.y;
        s.oz[p] = point.z + sc.spawn_eps * nd.z;
        s.dx[p] = nd.x; s.dy[p] = nd.y; s.dz[p] = nd.z;
        if (fmax(fmax(T[0], T[1]), T[2]) >= sc.threshold) next[reserve(next_n)] = p;
    }
}

// One thread per pixel of the chunk: A[row0 + pixel, face, :] += records in
// the reference's order (emitters.py:147-159 batches of `per_batch` samples
// of every pixel; per batch bounce 1..depth, samples in order; np.add.at is
// sequential). Paths of slot i are i * spp + s (k_raygen).
__global__ void k_transport_reduce(int64_t n_slots, int32_t spp, int32_t depth, int32_t per_batch,
                                   int32_t n_faces, const int32_t* __restrict__ rec_face,
                                   const double* __restrict__ rec_val, int64_t pixel_base,
                                   double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_slots;
         i += (int64_t)gridDim.x * blockDim.x) {
        double* row = out + (pixel_base + i) * (int64_t)n_faces * 3;
        for (int32_t s0 = 0; s0 < spp; s0 += per_batch) {
            const int32_t s1 = min(spp, s0 + per_batch);
            for (int32_t b = 0; b < depth; ++b)
                for (int32_t smp = s0; smp < s1; ++smp) {
                    const int64_t r = (i * spp + smp) * depth + b;
                    const int32_t f = rec_face[r];
                    if (f < 0) continue;
                    for (int ch = 0; ch < 3; ++ch) row[3 * f + ch] = row[3 * f + ch] + rec_val[3 * r + ch];
                }
        }
    }
}

__global__ void k_gather_L(Args a, double* out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < a.n_slots;
         p += (int64_t)gridDim.x * blockDim.x) {
        out[3 * p] = a.ps.Lr[p];
        out[3 * p + 1] = a.ps.Lg[p];
        out[3 * p + 2] = a.ps.Lb[p];
        if (!(isfinite(a.ps.Lr[p]) && isfinite(a.ps.Lg[p]) && isfinite(a.ps.Lb[p])))
            atomicAdd(&a.ps.counters[C_NONFINITE], 1);
    }
}

__global__ void k_reset_queue(int32_t* counters, int32_t which) {
    counters[which] = 0;
    counters[C_FETCH] = 0;
}

// Per-pixel sum over its spp paths in sample order, then / spp (render.py:348-350).
// Per-pixel sum in the reference's grouping (render.py:333-350): a 16-row
// band of npix = rows * w pixels is traced in batches of
// max(1, 65536 // npix) samples per pixel, each batch summed over its
// samples left to right (`L.reshape(npix, sb, 3).sum(axis=1)`, a sequential
// reduce in numpy), then added to the band's accumulator - so for frames
// wider than 4096 / spp the sums group exactly as the reference's do.
__global__ void k_accumulate(Args a) {
    const PathState& s = a.ps;
    const int64_t W = a.cam.width, H = a.cam.height;
    for (int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; slot < a.n_slots;
         slot += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pix = slot_pixel(a, slot);
        const int64_t row = pix / W, band = row - row % 16;
        const int64_t npix = min((int64_t)16, H - band) * W;
        const int32_t per_batch = (int32_t)max((int64_t)1, (int64_t)65536 / npix);
        double acc[3] = {0.0, 0.0, 0.0};
        for (int32_t k0 = 0; k0 < a.spp; k0 += per_batch) {
            const int32_t k1 = min(a.spp, k0 + per_batch);
            const int64_t p0 = slot * a.spp + k0;
            double b[3] = {s.Lr[p0], s.Lg[p0], s.Lb[p0]};
            for (int32_t k = k0 + 1; k < k1; ++k) {
                const int64_t p = slot * a.spp + k;
                b[0] = b[0] + s.Lr[p];
                b[1] = b[1] + s.Lg[p];
                b[2] = b[2] + s.Lb[p];
            }
            acc[0] = acc[0] + b[0];
            acc[1] = acc[1] + b[1];
            acc[2] = acc[2] + b[2];
        }
        // (out_by_pixel: a raster frame, possibly rank 0's mapped over NVLink - the
        // frame "gather" is these stores, issued as each chunk's pixels finish)
        const int64_t oi = (a.tiled || a.out_by_pixel) ? pix : a.out_offset + slot;
        HRT_ASSERT(oi >= 0 && (!(a.tiled || a.out_by_pixel) || oi < (int64_t)a.cam.width * a.cam.height),
                   "output pixel", oi, (int64_t)a.cam.width * a.cam.height);
        double* o = a.out + 3 * oi;
        bool bad = false;
        for (int ch = 0; ch < 3; ++ch) {
            const double v = acc[ch] / (double)a.spp;
            o[ch] = v;
            bad |= !(isfinite(v) && v >= 0.0);
        }
        if (bad) atomicAdd(&a.ps.counters[C_NONFINITE], 1);
    }
}

// ------------------------------------------------- field-seam kernels
// sample_batch(p, d) on arbitrary points through the field engine: prep
// converts world fp64 points to the engine's field-frame fp32 batch, post
// masks vacuum / empty-cell samples (evaluated = 0).
__global__ void k_field_prep(DevField fld, const double* __restrict__ pts,
                             const double* __restrict__ dirs, int64_t n, int32_t use_occupancy,
                             int32_t field_frame, fws::SampleIn* in, float4* dir32, int32_t* ev) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const d3 pw = mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        const d3 pf = field_frame ? pw : field_point(fld, pw);
        bool e = inside_box(fld.lo, fld.hi, pf);
        if (e && use_occupancy) {
            int32_t c3[3];
            e = nerf::occ_test(fld.nf, nerf::occ_cell(fld.nf, pf, c3));
        }
        fws::SampleIn r;
        const float3 p32 = nerf::to_f32(pf);
        r.x = p32.x; r.y = p32.y; r.z = p32.z;
        r.path = e ? (int32_t)i : -1;      // the engine evaluates inside (occupied) points only
        in[i] = r;
        if (dirs) {
            const d3 df = field_dir(fld, mk(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]));
            dir32[i] = make_float4((float)df.x, (float)df.y, (float)df.z, 0.f);
        }
        ev[i] = e ? 1 : 0;
    }
}

__global__ void k_field_post(const float4* __restrict__ res, const int32_t* __restrict__ ev,
                             int64_t n, float* sigma, float* rgb) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 r = res[i];
        const bool e = ev[i] != 0;
        sigma[i] = e ? r.x : 0.f;
        if (rgb) {
            rgb[3 * i] = e ? r.y : 0.f;
            rgb[3 * i + 1] = e ? r.z : 0.f;
            rgb[3 * i + 2] = e ? r.w : 0.f;
        }
    }
}

template <int E, int F>
__global__ void k_field_encode(DevField fld, const double* __restrict__ pts, int64_t n, float* feat,
                               uint32_t* index) {
    const NeuralField& nf = fld.nf;
    constexpr int L = E / F;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const d3 pf = field_point(fld, mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
        const float3 rel = nerf::rel_coord(nf, pf);
        for (int l = 0; l < L; ++l) {
            float v[4];
            nerf::encode_level<F>(nf, nf.lv[l], rel, v);
            for (int j = 0; j < F; ++j) feat[i * E + l * F + j] = v[j];
            if (index) {
                const nerf::LevelCoord lc = nerf::level_coord(nf.lv[l], rel);
                for (int c = 0; c < 8; ++c)
                    index[(i * L + l) * 8 + c] = nerf::corner_index(nf.lv[l], lc, c, nf.tmask);
            }
        }
    }
}

// Occupancy bits from sigma at cell centres (P4): bit set iff sigma > thr.
__global__ void k_occ_bits(const float* sigma, int64_t n_cells, double thr, uint32_t* bits) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w * 32 >= n_cells) return;
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t c = w * 32 + b;
        if (c < n_cells && (double)sigma[c] > thr) word |= 1u << b;
    }
    bits[w] = word;
}

// --------------------------------------------------- parity probes (K1/K2)
__global__ void k_uniform(const int64_t* keys, int64_t n, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t* k = keys + 6 * i;
        out[i] = rng::uniform((uint64_t)k[0], k[1], k[2], k[3], k[4], k[5]);
    }
}

__global__ void k_primary(path::Camera cam, const int64_t* pix, const int64_t* smp, int64_t n,
                          uint64_t seed, int32_t strat, double* o, double* d) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        d3 oo, dd;
        path::primary_ray(cam, pix[i], smp[i], seed, strat, oo, dd);
        o[3 * i] = oo.x; o[3 * i + 1] = oo.y; o[3 * i + 2] = oo.z;
        d[3 * i] = dd.x; d[3 * i + 1] = dd.y; d[3 * i + 2] = dd.z;
    }
}

__global__ void k_rays(DevBvh b, const double* o, const double* d, const double* tmin,
                       const double* tmax, int64_t n, int32_t any, double* t_out, int64_t* f_out,
                       uint8_t* hit_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const d3 oo = mk(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
        const d3 dd = mk(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
        const double t0 = tmin ? tmin[i] : 0.0, t1 = tmax ? tmax[i] : INFINITY;
        if (any) {
            hit_out[i] = bvh::occluded(b, oo, dd, t0, t1) ? 1 : 0;
        } else {
            double t;
            const int32_t f = bvh::nearest(b, oo, dd, t0, t1, t);
            t_out[i] = t;
            f_out[i] = f;
        }
    }
}

}  // namespace kern
