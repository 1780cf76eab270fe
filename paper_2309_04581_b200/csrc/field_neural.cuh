// field_neural.cuh - the neural field's building blocks (SURVEY Appendix B
// P1-P4; CPU definition in oracle/field.py): hash-grid level coordinates,
// corner indices and the two-phase gather/accumulate the field engine
// (field_ws.cuh) runs per level, SH(16), output activations, occupancy
// lookups, and the packed-weight layout of the tcgen05 MLP.
#pragma once
#include <cuda_fp16.h>
#include "common.cuh"
#include "umma.cuh"

namespace nerf {

constexpr uint32_t kHashY = 2654435761u, kHashZ = 805459861u;

// Byte offsets of the packed layers inside NeuralField::wpack (host packs
// the same layout, api.cu pack_weights()).
struct WOff { uint32_t d1, d2, c1, c2, c3, total; };
__host__ __device__ constexpr WOff woff(int E) {
    return {0u, (uint32_t)(64 * E * 2), (uint32_t)(64 * E * 2 + 2048),
            (uint32_t)(64 * E * 2 + 2048 + 4096), (uint32_t)(64 * E * 2 + 2048 + 4096 + 8192),
            (uint32_t)(64 * E * 2 + 2048 + 4096 + 8192 + 2048)};
}

// ------------------------------------------------------------- encode (K5)
HRT_DEV float3 to_f32(d3 p) { return make_float3((float)p.x, (float)p.y, (float)p.z); }

struct LevelCoord {
    int32_t i[3];
    float f[3];
};

HRT_DEV LevelCoord level_coord(const NeuralLevel& lv, float3 rel) {
    LevelCoord c;
    const float x[3] = {__fmul_rn(rel.x, lv.scale[0]), __fmul_rn(rel.y, lv.scale[1]),
                        __fmul_rn(rel.z, lv.scale[2])};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int32_t i = (int32_t)floorf(x[a]);
        i = max(0, min(i, lv.n - 1));
        c.i[a] = i;
        c.f[a] = __fsub_rn(x[a], (float)i);
    }
    return c;
}

HRT_DEV uint32_t corner_index(const NeuralLevel& lv, const LevelCoord& c, int corner, uint32_t tmask) {
    const uint32_t X = (uint32_t)c.i[0] + (corner & 1);
    const uint32_t Y = (uint32_t)c.i[1] + ((corner >> 1) & 1);
    const uint32_t Z = (uint32_t)c.i[2] + (corner >> 2);
    if (lv.dense) return X + lv.r * Y + lv.r * lv.r * Z;
    return (X ^ (Y * kHashY) ^ (Z * kHashZ)) & tmask;
}


// acc (two packed fp32) = fma(w, v, acc) per lane of the pair: one FFMA2.
// (a.x * b.x, a.y * b.y), each rounded as a scalar FMUL: one FMUL2.
HRT_DEV float2 mul2(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&r);
}

HRT_DEV void fma2(float2& acc, float w, float2 v) {
    unsigned long long a = *reinterpret_cast<unsigned long long*>(&acc);
    const unsigned long long b = *reinterpret_cast<const unsigned long long*>(&v);
    unsigned long long ww;
    asm("mov.b64 %0, {%1, %1};" : "=l"(ww) : "f"(w));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(ww), "l"(b));
    acc = *reinterpret_cast<float2*>(&a);
}

// Gather the 8 corner entries of one level and accumulate them as two
// fma chains acc_x = fma(w, v, acc_x) from +0 over the corners with
// cx = x in corner order, feature = acc_0 + acc_1 (oracle/field.py
// neural_encode, pinned by glibc fmaf in oracle/native.c; the split lets the
// field engine give the two x halves to the two lanes of a pair). For F = 2, x-adjacent corners
// whose entries form an aligned 16-byte pair (idx(c+1) == idx(c) ^ 1) are
// fetched with one float4 load; level bases are 16-byte aligned (hrt.cu pads
// level offsets).
template <int F>
HRT_DEV void gather_accumulate(const float* __restrict__ lvl_base, const uint32_t idx[8],
                               const float w[8], float* out) {
    if constexpr (F == 2) {
        const float2* base = reinterpret_cast<const float2*>(lvl_base);
        float2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(base + idx[k]);
        float2 acc[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
        for (int k = 0; k < 8; ++k) fma2(acc[k & 1], w[k], v[k]);
        out[0] = __fadd_rn(acc[0].x, acc[1].x);
        out[1] = __fadd_rn(acc[0].y, acc[1].y);
    } else {
        const float4* base = reinterpret_cast<const float4*>(lvl_base);
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(base + idx[k]);
        float2 a0[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
        float2 a1[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            fma2(a0[k & 1], w[k], make_float2(v[k].x, v[k].y));
            fma2(a1[k & 1], w[k], make_float2(v[k].z, v[k].w));
        }
        out[0] = __fadd_rn(a0[0].x, a0[1].x); out[1] = __fadd_rn(a0[0].y, a0[1].y);
        out[2] = __fadd_rn(a1[0].x, a1[1].x); out[3] = __fadd_rn(a1[0].y, a1[1].y);
    }
}

// One level of the encoding, F = 2 or 4 features. Dense and hashed levels
// take separate (warp-uniform) branches; the per-axis hash products are
// formed once ((Y+1)*P == Y*P + P in uint32) and the corner weights share
// their x*y products, with the oracle's rounding order ((wx*wy)*wz).
template <int F>
HRT_DEV void encode_level(const NeuralField& nf, const NeuralLevel& lv, float3 rel, float* out) {
    const LevelCoord c = level_coord(lv, rel);
    const float gx = __fsub_rn(1.0f, c.f[0]), gy = __fsub_rn(1.0f, c.f[1]),
                gz = __fsub_rn(1.0f, c.f[2]);
    const float wxy[4] = {__fmul_rn(gx, gy), __fmul_rn(c.f[0], gy), __fmul_rn(gx, c.f[1]),
                          __fmul_rn(c.f[0], c.f[1])};
    float w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = __fmul_rn(wxy[k & 3], (k & 4) ? c.f[2] : gz);
    const float* lvl_base = nf.table + (size_t)lv.offset * F;
    const uint32_t X = (uint32_t)c.i[0], Y = (uint32_t)c.i[1], Z = (uint32_t)c.i[2];
    uint32_t idx[8];
    if (lv.dense) {
        const uint32_t r = lv.r, rr = r * r;
        const uint32_t b0 = X + r * Y + rr * Z;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            idx[k] = b0 + (uint32_t)(k & 1) + ((k & 2) ? r : 0u) + ((k & 4) ? rr : 0u);
        gather_accumulate<F>(lvl_base, idx, w, out);
    } else {
        const uint32_t hy0 = Y * kHashY, hy1 = hy0 + kHashY;
        const uint32_t hz0 = Z * kHashZ, hz1 = hz0 + kHashZ;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            idx[k] = ((X + (uint32_t)(k & 1)) ^ ((k & 2) ? hy1 : hy0) ^ ((k & 4) ? hz1 : hz0)) & nf.tmask;
        gather_accumulate<F>(lvl_base, idx, w, out);
    }
}

// Two-phase form of a level for the field engine: level_issue() computes the
// corner indices and starts the 8 loads, level_finish() forms the weights and
// accumulates (same arithmetic, same order as encode_level), so two levels of
// gathers can be in flight per thread.
template <int F> struct FVec { using T = float2; };
template <> struct FVec<4> { using T = float4; };

template <int F>
struct LevelLoadsF {
    LevelCoord c;
    typename FVec<F>::T v[8];
};
using LevelLoads = LevelLoadsF<2>;

// Hashed levels start on a multiple of T entries in the device table
// (hrt.cu setup_field), so the physical entry off + ((X ^ hY ^ hZ) & mask)
// equals (X & mask) ^ (hY & mask) ^ ((hZ & mask) | off): per level the six
// masked terms are formed once, per corner one 3-input XOR (LOP3) gives the
// texel / element index.
template <int F = 2>
HRT_DEV void level_issue(const NeuralField& nf, const NeuralLevel& lv, float3 rel, LevelLoadsF<F>& g,
                         bool tex_level = false) {
    using V = typename FVec<F>::T;
    g.c = level_coord(lv, rel);
    const V* tab = reinterpret_cast<const V*>(nf.table);
    const uint32_t X = (uint32_t)g.c.i[0], Y = (uint32_t)g.c.i[1], Z = (uint32_t)g.c.i[2];
    const uint32_t off = (uint32_t)lv.offset;
    if (lv.dense) {
        const uint32_t r = lv.r, rr = r * r;
        const uint32_t b0 = off + X + r * Y + rr * Z;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            g.v[k] = __ldg(tab + (b0 + (uint32_t)(k & 1) + ((k & 2) ? r : 0u) + ((k & 4) ? rr : 0u)));
    } else {
        const uint32_t m = nf.tmask;
        const uint32_t hy = Y * kHashY, hz = Z * kHashZ;
        const uint32_t xs[2] = {X & m, (X + 1u) & m};
        const uint32_t ys[2] = {hy & m, (hy + kHashY) & m};
        const uint32_t zs[2] = {(hz & m) | off, ((hz + kHashZ) & m) | off};
        if (tex_level) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                g.v[k] = tex1Dfetch<V>(nf.tex, (int)(xs[k & 1] ^ ys[(k >> 1) & 1] ^ zs[k >> 2]));
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) g.v[k] = __ldg(tab + (xs[k & 1] ^ ys[(k >> 1) & 1] ^ zs[k >> 2]));
        }
    }
}

#ifndef HRT_PACKED_WEIGHTS
#define HRT_PACKED_WEIGHTS 1
#endif
template <int F = 2>
HRT_DEV void level_finish(const LevelLoadsF<F>& g, float* out) {
    const LevelCoord& c = g.c;
    const float gx = __fsub_rn(1.0f, c.f[0]), gy = __fsub_rn(1.0f, c.f[1]),
                gz = __fsub_rn(1.0f, c.f[2]);
    // wxy = (gx gy, fx gy, gx fy, fx fy); corner k weight = wxy[k & 3] * (gz | fz),
    // formed as FMUL2 pairs (each lane rounded as a scalar FMUL)
    float wxy[4], w[8];
    if (HRT_PACKED_WEIGHTS) {
        const float2 x2 = make_float2(gx, c.f[0]);
        const float2 a = mul2(x2, make_float2(gy, gy)), b = mul2(x2, make_float2(c.f[1], c.f[1]));
        wxy[0] = a.x; wxy[1] = a.y; wxy[2] = b.x; wxy[3] = b.y;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 p = mul2(make_float2(wxy[k], wxy[k]), make_float2(gz, c.f[2]));
            w[k] = p.x;
            w[k + 4] = p.y;
        }
    } else {
        wxy[0] = __fmul_rn(gx, gy); wxy[1] = __fmul_rn(c.f[0], gy);
        wxy[2] = __fmul_rn(gx, c.f[1]); wxy[3] = __fmul_rn(c.f[0], c.f[1]);
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = __fmul_rn(wxy[k & 3], (k & 4) ? c.f[2] : gz);
    }
    if constexpr (F == 2) {
        float2 acc[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
        for (int k = 0; k < 8; ++k) fma2(acc[k & 1], w[k], g.v[k]);
        out[0] = __fadd_rn(acc[0].x, acc[1].x);
        out[1] = __fadd_rn(acc[0].y, acc[1].y);
    } else {
        // same chains as gather_accumulate<4>: features (0,1) and (2,3) as FFMA2 pairs
        float2 a0[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
        float2 a1[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            fma2(a0[k & 1], w[k], make_float2(g.v[k].x, g.v[k].y));
            fma2(a1[k & 1], w[k], make_float2(g.v[k].z, g.v[k].w));
        }
        out[0] = __fadd_rn(a0[0].x, a0[1].x); out[1] = __fadd_rn(a0[0].y, a0[1].y);
        out[2] = __fadd_rn(a1[0].x, a1[1].x); out[3] = __fadd_rn(a1[0].y, a1[1].y);
    }
}

HRT_DEV float3 rel_coord(const NeuralField& nf, d3 pf) {
    const float3 p = to_f32(pf);
    return make_float3(__fsub_rn(p.x, nf.lo32[0]), __fsub_rn(p.y, nf.lo32[1]),
                       __fsub_rn(p.z, nf.lo32[2]));
}

// ------------------------------------------------------------ occupancy
HRT_DEV int32_t occ_cell(const NeuralField& nf, d3 pf, int32_t c[3]) {
    const float3 rel = rel_coord(nf, pf);
    const float x[3] = {__fmul_rn(rel.x, nf.occ_scale[0]), __fmul_rn(rel.y, nf.occ_scale[1]),
                        __fmul_rn(rel.z, nf.occ_scale[2])};
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = max(0, min((int32_t)floorf(x[a]), nf.occ_res - 1));
    return c[0] + nf.occ_res * (c[1] + nf.occ_res * c[2]);
}

HRT_DEV bool occ_test(const NeuralField& nf, int32_t cell) {
    return (__ldg(nf.occ + (cell >> 5)) >> (cell & 31)) & 1u;
}

// --------------------------------------------------------------- SH (P3)
HRT_DEV void sh16(float x, float y, float z, float* o) {
    const float xx = x * x, yy = y * y, zz = z * z;
    o[0] = 0.28209479177387814f;
    o[1] = -0.4886025119029199f * y;
    o[2] = 0.4886025119029199f * z;
    o[3] = -0.4886025119029199f * x;
    o[4] = 1.0925484305920792f * x * y;
    o[5] = -1.0925484305920792f * y * z;
    o[6] = 0.31539156525252005f * (3.0f * zz - 1.0f);
    o[7] = -1.0925484305920792f * x * z;
    o[8] = 0.5462742152960396f * (xx - yy);
    o[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    o[10] = 2.890611442640554f * x * y * z;
    o[11] = -0.4570457994644658f * y * (5.0f * zz - 1.0f);
    o[12] = 0.3731763325901154f * z * (5.0f * zz - 3.0f);
    o[13] = -0.4570457994644658f * x * (5.0f * zz - 1.0f);
    o[14] = 1.445305721320277f * z * (xx - yy);
    o[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

HRT_DEV float out_act(float x, int act) {
    if (act == 0) return 1.0f / (1.0f + expf(-x));
    return x > 20.0f ? x : log1pf(expf(x));
}

}  // namespace nerf
