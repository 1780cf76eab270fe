/*
 * oracle/native.c - TEST INFRASTRUCTURE ONLY (CPU parity oracle).
 *
 * The one part of the reference path numpy cannot restate bit-exactly:
 * `Camera.primary_rays` (reference pkg/src/hybridrt/render.py:61-74) turns
 * camera-space directions into world space with `Transform.direction`
 * (core.py:183-187), a numpy `@` that OpenBLAS evaluates as the fused chain
 * fma(x2, r2, fma(x1, r1, x0 * r0)) per output row (re-verified
 * against the reference in tests/test_oracle_reference.py). glibc's fma()
 * is correctly rounded, so this file pins that order exactly.
 *
 * Never linked into the product; built into oracle/_build/ by build().
 */
#include <math.h>
#include <stdint.h>

/* d_out[3*i+r] = fma(v2, R[r][2], fma(v1, R[r][1], v0 * R[r][0])) */
void oracle_rotate_fma(int64_t n, const double *v, const double *rot, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        const double *x = v + 3 * i;
        for (int r = 0; r < 3; ++r) {
            const double *row = rot + 3 * r;
            out[3 * i + r] = fma(x[2], row[2], fma(x[1], row[1], x[0] * row[0]));
        }
    }
}

/*
 * Hash-grid corner accumulation of the neural field (definition in
 * oracle/field.py): per sample and feature, two chains
 * acc_x = fmaf(w_c, v_c, acc_x) over the corners c with c & 1 == x in
 * increasing c, from +0; feature = acc_0 + acc_1 (float add). fmaf is
 * correctly rounded, so this pins the GPU's fma.rn.f32x2 accumulation (and
 * its lane-pair split of the corners) bit for bit.
 *   w: n x 8, v: n x 8 x F, out: n x F (float32)
 */
void oracle_corner_fma(int64_t n, int32_t F, const float *w, const float *v, float *out)
{
    for (int64_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < F; ++j) {
            float acc[2] = {0.0f, 0.0f};
            for (int k = 0; k < 8; ++k)
                acc[k & 1] = fmaf(w[8 * i + k], v[(8 * i + k) * F + j], acc[k & 1]);
            out[i * F + j] = acc[0] + acc[1];
        }
}
