// probe.cuh - measurement kernel behind hrt_gather_peak: the roofline of the
// hash-grid encode. The encode is bound by random 8-byte gathers from the
// L2-resident table (ncu: L1 miss-request path ~87 % busy), so its peak is
// measured here on the same table: every thread issues independent gathers
// at pseudo-random entries (LSU or TEX path), 8 in flight.
#pragma once
#include "common.cuh"

namespace probe {

HRT_DEV uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; return x ^ (x >> 16);
}

template <bool kTex>
__global__ void __launch_bounds__(512) k_gather(const float2* __restrict__ table,
                                                 unsigned long long tex, uint32_t n_entries,
                                                 int32_t iters, float* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int32_t it = 0; it < iters; ++it) {
        float2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t idx = mix32(tid * 0x9E3779B9U + (uint32_t)(it * 8 + u)) % n_entries;
            v[u] = kTex ? tex1Dfetch<float2>(tex, (int)idx) : __ldg(table + idx);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 1234.5f) sink[0] = acc;     // keep the loads alive
}

}  // namespace probe
