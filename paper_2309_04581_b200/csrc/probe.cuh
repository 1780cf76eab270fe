// probe.cuh - measurement kernel behind hrt_gather_peak: the roofline of the
// hash-grid encode. The encode is bound by random 8-byte gathers from the
// L2-resident table (ncu: L1 miss-request path ~87 % busy), so its peak is
// measured here on the same table: every thread issues independent gathers
// at pseudo-random entries (LSU or TEX path), 8 in flight, one table entry
// (8 B for F = 2, 16 B for F = 4) each.
#pragma once
#include "common.cuh"

namespace probe {

HRT_DEV uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; return x ^ (x >> 16);
}

// V = float2 (F = 2, 8-B entries) or float4 (F = 4, 16-B entries).
template <bool kTex, typename V>
__global__ void __launch_bounds__(512) k_gather(const V* __restrict__ table,
                                                 unsigned long long tex, uint32_t n_entries,
                                                 int32_t iters, float* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int32_t it = 0; it < iters; ++it) {
        V v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t idx = mix32(tid * 0x9E3779B9U + (uint32_t)(it * 8 + u)) % n_entries;
            v[u] = kTex ? tex1Dfetch<V>(tex, (int)idx) : __ldg(table + idx);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 1234.5f) sink[0] = acc;     // keep the loads alive
}

}  // namespace probe

namespace probe {

// L2 read roofline (hrt_l2_peak): every SM streams an L2-resident buffer
// (the hash table itself, after a warm pass) with coalesced 16-B loads.
__global__ void __launch_bounds__(512) k_l2_read(const uint4* __restrict__ buf, int64_t n16,
                                                  int32_t passes, float* sink) {
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int32_t p = 0; p < passes; ++p) {
        int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n16; i += 4 * stride) {
            const uint4 a = __ldcg(buf + i), b = __ldcg(buf + i + stride);
            const uint4 c = __ldcg(buf + i + 2 * stride), d = __ldcg(buf + i + 3 * stride);
            acc ^= a.x ^ b.y ^ c.z ^ d.w;
        }
        for (; i < n16; i += stride) acc ^= __ldcg(buf + i).x;
    }
    if (acc == 0x12345678u) sink[0] = (float)acc;
}

// Random whole-sector gathers: lane pairs read the two 16-B halves of one
// random 32-B sector of the buffer (16 sectors per warp instruction, L1
// bypassed), 8 instructions in flight per thread.
__global__ void __launch_bounds__(512) k_sector_gather(const uint4* __restrict__ buf, uint32_t n_sectors,
                                                        int32_t iters, float* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t half = tid & 1u;
    uint32_t acc = 0;
    for (int32_t it = 0; it < iters; ++it) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t s = mix32((tid >> 1) * 0x9E3779B9U + (uint32_t)(it * 8 + u)) % n_sectors;
            v[u] = __ldcg(buf + 2ull * s + half);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) sink[0] = (float)acc;
}

}  // namespace probe
