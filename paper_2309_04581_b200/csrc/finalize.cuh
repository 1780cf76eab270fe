// finalize.cuh - K9 output stage: the reference's finalize (render.py:399-401)
// on the device. PFM (images.py:37-40): little-endian float32 RGB, rows
// bottom-up; PPM P6 (images.py:59-64): sRGB tone map (core.py:51-64) then
// round-half-up 8-bit codes, rows top-down. Rows come either as a raster
// frame or as the gathered per-rank tile buffers with their global pixel ids
// (pixel < 0 = padding), so unpacking the multi-GPU gather and encoding are
// one pass over the frame.
#pragma once
#include "common.cuh"

namespace fin {

constexpr double kSrgbCut = 0.0031308;

// core.py:51-64 for one channel (finite input): 12.92 x below the cut,
// 1.055 x^(1/2.4) - 0.055 above, exactly 1 for x >= 1, clipped to [0, 1].
HRT_DEV double tone_map(double c) {
    const double lo = 12.92 * c;
    const double hi = 1.055 * pow(fmax(c, kSrgbCut), 1.0 / 2.4) - 0.055;
    double out = c <= kSrgbCut ? lo : hi;
    if (c >= 1.0) out = 1.0;
    return fmin(fmax(out, 0.0), 1.0);
}

__global__ void k_finalize(int32_t w, int32_t h, const double* __restrict__ src,
                           const int32_t* __restrict__ pixel, int64_t n, int32_t hdr, int64_t head,
                           uint8_t* __restrict__ out, int32_t* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = pixel ? (int64_t)pixel[i] : i;
        if (p < 0) continue;
        const int64_t x = p % w, y = p / w;
        for (int ch = 0; ch < 3; ++ch) {
            const double v = src[3 * i + ch];
            if (!hdr && !isfinite(v)) atomicAdd(bad, 1);   // tone_map asserts finite; PFM does not
            if (hdr) {
                const float f = (float)v;
                const uint32_t b = __float_as_uint(f);
                uint8_t* o = out + head + (((int64_t)(h - 1 - y) * w + x) * 3 + ch) * 4;
                o[0] = (uint8_t)b; o[1] = (uint8_t)(b >> 8); o[2] = (uint8_t)(b >> 16); o[3] = (uint8_t)(b >> 24);
            } else {
                const double s = isfinite(v) ? tone_map(v) : 0.0;
                out[head + (y * w + x) * 3 + ch] = (uint8_t)floor(s * 255.0 + 0.5);
            }
        }
    }
}

}  // namespace fin
