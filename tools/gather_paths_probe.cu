// Dev probe: random-gather throughput of the L2-resident hash table through
// the different SM load paths (LSU 8 B, LSU 16 B, TEX 8 B, TMA bulk 16 B into
// shared memory, and LSU + TMA side by side in one kernel). Answers whether
// the TMA unit reaches L2 past the L1TEX miss path that bounds the encode.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_gp tools/gather_paths_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; return x ^ (x >> 16);
}

template <int kBytes>
__global__ void __launch_bounds__(512) k_lsu(const char* __restrict__ tab, uint32_t n16, int iters, float* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t idx = mix32(tid * 0x9E3779B9U + (uint32_t)(it * 8 + u)) % n16;
            if (kBytes == 16) v[u] = __ldg(reinterpret_cast<const float4*>(tab) + idx);
            else { float2 t = __ldg(reinterpret_cast<const float2*>(tab) + 2 * idx); v[u] = make_float4(t.x, t.y, 0, 0); }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z;
    }
    if (acc == 1234.5f) sink[0] = acc;
}

// kGroup lanes share one random 128-B line and read kGroup different 32-B
// sectors of it (8 B each) in the same instruction: one L1 miss request with a
// sector mask, or kGroup requests?
template <int kGroup>
__global__ void __launch_bounds__(512) k_line(const char* __restrict__ tab, uint32_t n_lines, int iters, float* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t g = tid / kGroup, sub = tid % kGroup;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t line = mix32(g * 0x9E3779B9U + (uint32_t)(it * 8 + u)) % n_lines;
            v[u] = __ldg(reinterpret_cast<const float2*>(tab + 128ull * line + 32 * sub));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 1234.5f) sink[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
        :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk16(void* dst, const void* src, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                 :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src),
                    "r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}

// kMix: warps with (warp & 1) do LSU 8-B gathers instead of TMA.
template <int kPer, bool kMix>
__global__ void __launch_bounds__(512) k_tma(const char* __restrict__ tab, uint32_t n16, int iters, float* sink) {
    extern __shared__ __align__(16) char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);            // 2 per warp
    float4* buf = reinterpret_cast<float4*>(smem + 16 * nw);       // [warp][2][32*kPer]
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (lane == 0) { mbar_init(&bars[2 * warp], 32); mbar_init(&bars[2 * warp + 1], 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    float acc = 0.f;
    if (kMix && (warp & 1)) {
        for (int it = 0; it < iters * 2; ++it) {
            float2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t idx = mix32(tid * 0x9E3779B9U + (uint32_t)(it * 8 + u)) % (2 * n16);
                v[u] = __ldg(reinterpret_cast<const float2*>(tab) + idx);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
        }
    } else {
        float4* mine = buf + (size_t)warp * 2 * 32 * kPer;
        auto issue = [&](int it, int s) {
            mbar_expect(&bars[2 * warp + s], 16 * kPer);
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const uint32_t idx = mix32(tid * 0x9E3779B9U + (uint32_t)(it * kPer + u)) % n16;
                bulk16(&mine[(s * 32 + lane) * kPer + u], tab + 16ull * idx, &bars[2 * warp + s]);
            }
        };
        const int n_it = iters * 8 / kPer;
        issue(0, 0);
        for (int it = 0; it < n_it; ++it) {
            const int s = it & 1;
            if (it + 1 < n_it) issue(it + 1, s ^ 1);
            mbar_wait(&bars[2 * warp + s], (it >> 1) & 1);
#pragma unroll
            for (int u = 0; u < kPer; ++u) { float4 v = mine[(s * 32 + lane) * kPer + u]; acc += v.x + v.y; }
            __syncwarp();
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

int main() {
    const size_t bytes = 46.5 * 1024 * 1024;
    const uint32_t n16 = (uint32_t)(bytes / 16);
    char* tab; float* sink;
    cudaMalloc(&tab, bytes); cudaMalloc(&sink, 4);
    cudaMemset(tab, 0, bytes);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 64;
    auto time = [&](const char* name, auto launch, double reqs, double useful_b) {
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double s = ms * 1e-3 / 5;
        printf("%-28s %8.1f G req/s  %8.1f GB/s useful  (%s)\n", name, reqs / s / 1e9, reqs * useful_b / s / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int bpsm : {2, 4}) {
        const int blocks = sms * bpsm, thr = 512;
        const double reqs = (double)blocks * thr * iters * 8;
        printf("-- %d blocks/SM x 512 threads\n", bpsm);
        time("LSU 8B", [&] { k_lsu<8><<<blocks, thr>>>(tab, n16, iters, sink); }, reqs, 8);
        time("LSU 16B", [&] { k_lsu<16><<<blocks, thr>>>(tab, n16, iters, sink); }, reqs, 16);
        time("line x2 lanes (sectors)", [&] { k_line<2><<<blocks, thr>>>(tab, n16 / 8, iters, sink); }, reqs, 8);
        time("line x4 lanes (sectors)", [&] { k_line<4><<<blocks, thr>>>(tab, n16 / 8, iters, sink); }, reqs, 8);
        time("line x1 (sectors)", [&] { k_line<1><<<blocks, thr>>>(tab, n16 / 8, iters, sink); }, reqs, 8);
        const size_t sm4 = 16 * 16 + 16 * 2 * 32 * 4 * 16, sm8 = 16 * 16 + 16 * 2 * 32 * 8 * 16;
        cudaFuncSetAttribute(k_tma<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
        cudaFuncSetAttribute(k_tma<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8);
        cudaFuncSetAttribute(k_tma<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
        if (bpsm == 2) {
            time("TMA bulk 16B x4", [&] { k_tma<4, false><<<blocks, thr, sm4>>>(tab, n16, iters, sink); }, reqs, 16);
            time("TMA bulk 16B x8 (1 blk/SM)", [&] { k_tma<8, false><<<sms, thr, sm8>>>(tab, n16, iters, sink); },
                 (double)sms * thr * iters * 8, 16);
            // mixed: half the warps TMA (iters*8 reqs), half LSU 8B (iters*16 reqs)
            const double rq = (double)blocks * thr / 2 * iters * 8;
            // per unit time the LSU half issued 2*rq 8-B gathers: sectors = rq (16B TMA) + 2 rq (LSU)
            time("mixed: TMA16 + 2x LSU8 sectors", [&] { k_tma<4, true><<<blocks, thr, sm4>>>(tab, n16, iters, sink); }, 3 * rq, 8);
        }
    }
    return 0;
}
