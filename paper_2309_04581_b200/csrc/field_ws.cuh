// field_ws.cuh - warp-specialized NeRF field engine (K5 + K6) for batches of
// samples. The hash-grid encode and the tcgen05 MLP run in different warps,
// and every MMA A operand lives in TMEM, so the L1 data pipe carries only
// the table gathers (round-1 ncu: with A tiles in smem the pipe was 97 %
// busy, ~45 % of it shared-memory operand traffic).
//
// CTA (persistent, one per SM, 512 TMEM columns):
//   16 encode warps: warp w owns TMEM lanes 32*(w%4).. (= tile rows) and the
//       level quarter q = w/4; per tile it gathers levels [qL/4, (q+1)L/4) of
//       its 32 rows, packs fp16 pairs and tcgen05.st's them into the tile's
//       stage columns, then arrives on full[s].
//   1 MMA warp (one elected thread, no TMEM ld/st): per tile, waits full[s],
//       issues D1 with A = stage s in TMEM (commit frees the stage and
//       signals accf[g]), then D2, C1, C2, C3 with A = group g's activation
//       columns, each after the epilogue's actr[g] arrival.
//   2 epilogue groups x 4 warps (warp <-> lane quarter): group g = tile % 2
//       turns each accumulator into the next layer's fp16 A operand
//       (tcgen05.ld -> ReLU -> tcgen05.st) and writes (sigma, rgb).
// TMEM columns: stages [0, 4*E/2); group g: accum [128+128g, +64),
// activations [192+128g, +32). Weights (B operands) stay in smem.
// Numerics equal field_neural.cuh / oracle/field.py (same encode, fp16
// operands, fp32 accumulation).
#pragma once
#include <cuda_fp16.h>
#include "common.cuh"
#include "field_neural.cuh"
#include "umma.cuh"

namespace fws {

// HRT_WS_PROFILE builds accumulate per-role cycle counts into ws_prof
// (dev aid: [0] enc total, [1] enc wait-empty, [2] epi total, [3] epi
// wait-accf, [4] mma total, [5] mma wait-full, [6] mma wait-actr).
#ifdef HRT_WS_PROFILE
__device__ unsigned long long ws_prof[8];
#define WS_T0(v) const long long v = clock64()
#define WS_ADD(i, t0) atomicAdd(&ws_prof[i], (unsigned long long)(clock64() - (t0)))
#else
#define WS_T0(v)
#define WS_ADD(i, t0)
#endif

#ifndef HRT_WS_GROUPS
#define HRT_WS_GROUPS 2
#endif
#ifndef HRT_WS_STAGES
#define HRT_WS_STAGES 6
#endif
#ifndef HRT_WS_INFLIGHT
#define HRT_WS_INFLIGHT 2
#endif
#ifndef HRT_STREAM_OUT
#define HRT_STREAM_OUT 1
#endif
#ifndef HRT_SYNTH_ENCODE
#define HRT_SYNTH_ENCODE 0
#endif
constexpr bool kSynthEncode = HRT_SYNTH_ENCODE;   // measurement build: MLP fed without gathers
#ifndef HRT_SYNTH_MLP
#define HRT_SYNTH_MLP 0
#endif
// measurement build: encoded tiles are released without MMAs and every row
// gets (sigma, rgb) = (1, 0.5, 0.5, 0.5) - what the encode sustains alone
constexpr bool kSynthMlp = HRT_SYNTH_MLP;
constexpr int kEncWarps = 16;               // 4 level quarters x 4 lane quarters
// Encode teams (template T): with T = 2 the 16 encode warps form two teams
// of 8 (2 level halves x 4 lane quarters, one level of gathers in flight per
// thread) that take alternate tiles, so two tiles are in flight per SM.
// Measured per round (DESIGN 4.2): +5-7 % on the first, L1-coherent march
// rounds of a chunk, -1-3 % on the later incoherent ones, so the host runs
// T = 2 for the first kTeamRounds rounds only. Same per-level arithmetic:
// the features do not depend on T.
constexpr int kInflight = HRT_WS_INFLIGHT;  // levels of gathers in flight per encode thread
#ifndef HRT_WS_INFLIGHT4
#define HRT_WS_INFLIGHT4 1
#endif
template <int F>
constexpr int kInflightF = F == 2 ? kInflight : HRT_WS_INFLIGHT4;   // F = 4: 16-B gathers
constexpr int kMlpGroups = HRT_WS_GROUPS;
constexpr int kMlpWarps = 4 * kMlpGroups;
constexpr int kThreads = 32 * (kEncWarps + kMlpWarps + 1);   // + MMA issuer warp
constexpr int kMaxStages = 8;                 // barrier slots reserved per ring
// encoded-tile ring depth: HRT_WS_STAGES tiles of E/2 TMEM columns, within the
// 128 columns below the MLP groups' (measured on cfg1: 6 stages 1 % faster than 4)
template <int E>
constexpr int kStagesE = HRT_WS_STAGES * (E / 2) <= 128 ? HRT_WS_STAGES : 128 / (E / 2);
static_assert(HRT_WS_STAGES <= kMaxStages, "stage ring");
constexpr int kRows = 128;
constexpr uint32_t kTmemCols = 512;

// One sample of a batch: field-frame float32 position (exactly
// float(field_point(p)), the encode input) and the owning path id (SH
// direction lookup + composite bookkeeping).
struct __align__(16) SampleIn {
    float x, y, z;
    int32_t path;
};

// Logical batch row l -> physical row of the sample-major march batch: the
// batch of a round is `width` live paths x S samples laid out with row
// stride `stride` (the previous queue length), i.e. l -> (l / width) *
// stride + l % width; width == 0 is the identity (dense batches).
struct RowMap {
    int64_t stride;
    int32_t width;
    uint32_t magic;         // l / width == (l * magic) >> shift for l < 2^31 (set_rows)
    uint32_t shift;
};
// Device-driven rounds set the map from the round counters: the division by
// `width` becomes one wide multiply + shift (magic = ceil(2^s / width),
// s = 31 + ceil(log2 width); exact for l < 2^31 since l * (magic * width -
// 2^s) < 2^31 * width <= 2^s).
__device__ __forceinline__ void set_rows(RowMap& m, int32_t width, int64_t stride) {
    m.width = width;
    m.stride = stride;
    if (width <= 0) return;
    const uint32_t lg = width > 1 ? 32u - (uint32_t)__clz(width - 1) : 0u;
    m.shift = 31u + lg;
    m.magic = (uint32_t)(((1ull << m.shift) + (uint64_t)width - 1) / (uint64_t)width);
}
__device__ __forceinline__ int64_t phys_row(const RowMap& m, int64_t l) {
    if (m.width == 0) return l;
    const uint32_t i = (uint32_t)(((uint64_t)(uint32_t)l * m.magic) >> m.shift);   // l / width
    return (int64_t)i * m.stride + (int64_t)((uint32_t)l - i * (uint32_t)m.width);
}

struct SmemPlan {
    uint32_t w, bars, tslot, total;
};
__host__ __device__ constexpr SmemPlan plan(int E) {
    return {0u, nerf::woff(E).total, nerf::woff(E).total + 256u, nerf::woff(E).total + 272u};
}

// barrier slots (8 B each): full[kMaxStages] (encoders -> MMA), empty[kMaxStages]
// (MMA commit -> encoders), accf[g] (MMA commit -> epilogue g), actr[g]
// (epilogue g -> MMA: activations written / accumulator consumed)
__device__ __forceinline__ uint32_t bar_full(uint32_t base, int s) { return base + 8u * s; }
__device__ __forceinline__ uint32_t bar_empty(uint32_t base, int s) { return base + 8u * (kMaxStages + s); }
__device__ __forceinline__ uint32_t bar_accf(uint32_t base, int g) { return base + 8u * (2 * kMaxStages + g); }
__device__ __forceinline__ uint32_t bar_actr(uint32_t base, int g) {
    return base + 8u * (2 * kMaxStages + kMlpGroups + g);
}

__device__ __forceinline__ void arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// D = A(TMEM, 128 x K) * B(smem, N x K)^T as K/16 UMMAs.
__device__ __forceinline__ void issue_ts(uint32_t tmem_d, uint32_t tmem_a, int K, uint32_t b_addr,
                                         int N) {
    const uint32_t id = umma::idesc_f16(kRows, N);
    for (int s = 0; s < K / 16; ++s)
        umma::mma_f16_ts(tmem_d, tmem_a + 8u * s, umma::desc(b_addr + 256u * s, K * 16), id,
                         s > 0 ? 1u : 0u);
}

// 64-wide layer epilogue: accum -> ReLU -> fp16 pairs -> activation columns.
__device__ __forceinline__ void relu64_tmem(uint32_t accum, uint32_t act) {
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16];
        umma::ld16(accum + c0, v);
        uint32_t h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = umma::pack_half2_relu(v[2 * i], v[2 * i + 1]);
        umma::st<8>(act + c0 / 2, h);
    }
    umma::wait_st();
}

// Batch evaluation of n samples -> out[i] = (sigma, r, g, b).
// dir32[path] is the field-frame unit direction; density_only skips the
// colour head (rgb = 0).
template <int E, int F, int T = 1>
__global__ void __launch_bounds__(kThreads, 1)
k_field_ws(NeuralField nf, const SampleIn* __restrict__ in, RowMap rmap, int64_t n,
           const float4* __restrict__ dir32, float4* __restrict__ out, int32_t density_only,
           const int32_t* __restrict__ round_ctr, unsigned long long* stats, int64_t* round_log) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr SmemPlan P = plan(E);
    constexpr nerf::WOff W = nerf::woff(E);
    constexpr int L = E / F;
    constexpr int LG = 4 / T;                     // level groups per team
    constexpr int NL = L / LG;                    // levels per encode thread
    constexpr int NC = NL * F / 2;                // TMEM columns per encode thread
    constexpr uint32_t kStageCols = E / 2;
    constexpr int kStages = kStagesE<E>;
    const int warp = threadIdx.x >> 5;
    if (round_ctr) {                 // device-driven march round (kern::k_round_begin counters)
        set_rows(rmap, round_ctr[C_MQ0 + (round_ctr[C_CUR] ^ 1)], round_ctr[C_STRIDE]);
        n = (int64_t)rmap.width * round_ctr[C_S];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (stats) atomicAdd(stats + S_ROWS, (unsigned long long)n);
            const int32_t ri = round_ctr[C_RIDX] - 1;                  // (k_round_begin's ordinal)
            if (round_log && ri >= 0 && ri < 1024) round_log[ri] = n;  // hrt_round_rows
        }
    }
    if (n <= 0) return;              // empty round: skip the prologue
    const int64_t tiles = (n + kRows - 1) / kRows;

    // ---- prologue: weights to smem, barriers, TMEM
    {
        const uint4* src = reinterpret_cast<const uint4*>(nf.wpack);
        uint4* dst = reinterpret_cast<uint4*>(smem + P.w);
        for (uint32_t i = threadIdx.x; i < W.total / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    const uint32_t bars = umma::saddr(smem + P.bars);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + P.tslot);
    if (warp == kEncWarps + kMlpWarps) umma::tmem_alloc(umma::saddr(tslot), kTmemCols);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            umma::mbar_init(bar_full(bars, s), kEncWarps / T * 32);   // one team fills a stage
            umma::mbar_init(bar_empty(bars, s), 1);
        }
        for (int g = 0; g < kMlpGroups; ++g) {
            umma::mbar_init(bar_accf(bars, g), 1);
            umma::mbar_init(bar_actr(bars, g), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;   // this warp's TMEM lane quarter

    WS_T0(t_role);
    if (warp < kEncWarps) {
        // ================= encode warps =================
        // (one code path for all level quarters: warps of all four quarters
        // share each scheduler, and four specialised copies of this loop
        // thrash the instruction cache - measured 1.9x slower)
        const int q = (warp >> 2) % LG;             // level group
        const int team = (warp >> 2) / LG;
        const int r = (warp & 3) * 32 + (threadIdx.x & 31);   // row == TMEM lane
        const float3 lo = make_float3(nf.lo32[0], nf.lo32[1], nf.lo32[2]);
        int it = team;
        for (int64_t t = blockIdx.x + (int64_t)team * gridDim.x; t < tiles;
             t += (int64_t)T * gridDim.x, it += T) {
            const int s = it % kStages;
            const uint32_t ph = (uint32_t)((it / kStages) & 1);
            const int64_t l = t * kRows + r;
            const int64_t i = l < n ? phys_row(rmap, l) : 0;
            float v[NL * F];
            const SampleIn si = l < n ? in[i] : SampleIn{0.f, 0.f, 0.f, -1};
            if (si.path >= 0) {
                const float3 rel = make_float3(__fsub_rn(si.x, lo.x), __fsub_rn(si.y, lo.y),
                                               __fsub_rn(si.z, lo.z));
                if constexpr (kSynthEncode) {
                    // measurement build only: features from the position, no table
                    // gathers - what the MLP pipeline sustains when it is fed
#pragma unroll
                    for (int k = 0; k < NL * F; ++k) v[k] = 0.01f * (float)k * rel.x - rel.y;
                } else if constexpr (NL % (T >= 2 ? 1 : kInflightF<F>) == 0) {
                    // kInflightF levels of gathers in flight per thread (1 with two teams)
                    constexpr int IF = T >= 2 ? 1 : kInflightF<F>;
#pragma unroll
                    for (int j = 0; j < NL; j += IF) {
                        nerf::LevelLoadsF<F> g[IF];
#pragma unroll
                        for (int u = 0; u < IF; ++u)
                            nerf::level_issue<F>(nf, nf.lv[q * NL + j + u], rel, g[u],
                                                 q * NL + j + u >= nf.tex_from);
#pragma unroll
                        for (int u = 0; u < IF; ++u) nerf::level_finish<F>(g[u], v + (j + u) * F);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < NL; ++j)
                        nerf::encode_level<F>(nf, nf.lv[q * NL + j], rel, v + j * F);
                }
            } else {
#pragma unroll
                for (int k = 0; k < NL * F; ++k) v[k] = 0.f;
            }
            uint32_t h[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) h[k] = umma::pack_half2(v[2 * k], v[2 * k + 1]);
            // stage free? (the gathers above already overlapped the wait)
            WS_T0(tw);
            if (it >= kStages) umma::mbar_wait(bar_empty(bars, s), ph ^ 1u);
            if ((threadIdx.x & 31) == 0) WS_ADD(1, tw);
            __syncwarp();
            umma::fence_after();
            umma::st<NC>(tmem + lane + (uint32_t)s * kStageCols + (uint32_t)(q * NC), h);
            umma::wait_st();
            umma::fence_before();
            arrive(bar_full(bars, s));
        }
    } else if (warp < kEncWarps + kMlpWarps) {
        // ================= epilogue groups =================
        // Group g owns tiles j with j % kMlpGroups == g. Per layer: wait the
        // accumulator (accf[g]), tcgen05.ld, activation, tcgen05.st the next
        // A operand, then arrive actr[g] (also "accumulator consumed").
        const int ew = warp - kEncWarps;
        const int g = ew / 4;
        const int m = (ew % 4) * 32 + (threadIdx.x & 31);   // row == TMEM lane
        const uint32_t accum = tmem + 128u + 128u * g + lane;
        const uint32_t act = accum + 64u;
        const uint32_t accf = bar_accf(bars, g), actr = bar_actr(bars, g);
        uint32_t aph = 0;
        auto take = [&]() {
            WS_T0(tw);
            umma::mbar_wait(accf, aph);
            if ((threadIdx.x & 31) == 0) WS_ADD(3, tw);
            aph ^= 1u;
            __syncwarp();
            umma::fence_after();
        };
        auto give = [&]() {
            umma::fence_before();
            arrive(actr);
        };
        int it = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
            if ((it % kMlpGroups) != g) continue;
            if constexpr (kSynthMlp) {
                const int64_t l = t * kRows + m;
                if (l < n) {
                    const int64_t i = phys_row(rmap, l);
                    if (in[i].path >= 0) __stcs(out + i, make_float4(1.f, .5f, .5f, .5f));
                }
                continue;
            }
            const int64_t l = t * kRows + m;
            const int64_t i = l < n ? phys_row(rmap, l) : 0;
            float3 dir = make_float3(0.f, 0.f, 1.f);
            const int32_t path = l < n ? in[i].path : -1;
            if (path >= 0 && !density_only) {
                const float4 d4 = dir32[path];
                dir = make_float3(d4.x, d4.y, d4.z);
            }
            take();                                         // D1 done
            relu64_tmem(accum, act);
            give();
            take();                                         // D2 done
            float o[16];
            umma::ld16(accum, o);
            const float sigma = expf(o[0]);
            float rgb[3] = {0.f, 0.f, 0.f};
            if (!density_only) {
                float c[32];
                nerf::sh16(dir.x, dir.y, dir.z, c);
#pragma unroll
                for (int k = 1; k < 16; ++k) c[15 + k] = o[k];
                c[31] = 0.0f;
                uint32_t hc[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) hc[k] = umma::pack_half2(c[2 * k], c[2 * k + 1]);
                umma::st<16>(act, hc);
                umma::wait_st();
                give();
                take();                                     // C1 done
                relu64_tmem(accum, act);
                give();
                take();                                     // C2 done
                relu64_tmem(accum, act);
                give();
                take();                                     // C3 done
                umma::ld16(accum, o);
                rgb[0] = nerf::out_act(o[0], nf.act);
                rgb[1] = nerf::out_act(o[1], nf.act);
                rgb[2] = nerf::out_act(o[2], nf.act);
            }
            give();                                         // accumulator free
            if (path >= 0) {
                const float4 o4 = make_float4(sigma, rgb[0], rgb[1], rgb[2]);
                if (HRT_STREAM_OUT) __stcs(out + i, o4);      // read once by k_step (evict-first)
                else out[i] = o4;
            }
        }
    } else if ((threadIdx.x & 31) == 0) {
        // ================= MMA issuer (one thread) =================
        // Walks tile pairs (one per group) layer by layer so one group's MMA
        // overlaps the other group's epilogue.
        const uint32_t wb = umma::saddr(smem + P.w);
        const int nl = kSynthMlp ? 1 : (density_only ? 2 : 5);
        const uint32_t boff[5] = {W.d1, W.d2, W.c1, W.c2, W.c3};
        const int kdim[5] = {E, 64, 32, 64, 64};
        const int ndim[5] = {64, 16, 64, 64, 16};
        int64_t J = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) ++J;
        uint32_t rph[kMlpGroups] = {};
        bool fresh[kMlpGroups];
        for (int g = 0; g < kMlpGroups; ++g) fresh[g] = true;
        for (int64_t j0 = 0; j0 < J; j0 += kMlpGroups) {
            for (int k = 0; k < nl; ++k) {
                for (int g = 0; g < kMlpGroups && j0 + g < J; ++g) {
                    const int64_t j = j0 + g;
                    const uint32_t accum = tmem + 128u + 128u * g;
                    const uint32_t actr = bar_actr(bars, g);
                    uint32_t a_src;
                    if (k == 0) {
                        const int s = (int)(j % kStages);
                        WS_T0(tf);
                        umma::mbar_wait(bar_full(bars, s), (uint32_t)((j / kStages) & 1));
                        WS_ADD(5, tf);
                        if constexpr (kSynthMlp) {
                            umma::fence_after();
                            arrive(bar_empty(bars, s));
                            continue;
                        }
                        WS_T0(ta);
                        if (!fresh[g]) { umma::mbar_wait(actr, rph[g]); rph[g] ^= 1u; }
                        WS_ADD(6, ta);
                        fresh[g] = false;
                        a_src = tmem + (uint32_t)s * kStageCols;
                    } else {
                        WS_T0(ta);
                        umma::mbar_wait(actr, rph[g]);
                        WS_ADD(6, ta);
                        rph[g] ^= 1u;
                        a_src = accum + 64u;
                    }
                    umma::fence_after();
                    issue_ts(accum, a_src, kdim[k], wb + boff[k], ndim[k]);
                    if (k == 0) umma::commit(bar_empty(bars, (int)(j % kStages)));
                    umma::commit(bar_accf(bars, g));
                }
            }
        }
    }
#ifdef HRT_WS_PROFILE
    if ((threadIdx.x & 31) == 0)
        WS_ADD(warp < kEncWarps ? 0 : (warp < kEncWarps + kMlpWarps ? 2 : 4), t_role);
#endif
    umma::fence_before();
    __syncthreads();
    if (warp == kEncWarps + kMlpWarps) umma::tmem_free(tmem, kTmemCols);
}

}  // namespace fws
