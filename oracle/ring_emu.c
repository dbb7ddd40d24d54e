/* O6 ring-order emulation — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain single-threaded C, compiled with -O2 -ffp-contract=off, no SIMD, sharing nothing with the
 * CUDA path.  It replays the order in which a ring allreduce (§2.2) adds the contributions of
 * the P workers to each element, with the n_r/Σn weights of Eq. 1 applied to each
 * contribution exactly once, at the hop where it enters the ring:
 *
 *   chunk c = [c·cs, min((c+1)·cs, count))       (cs: chunk size in elements, DESIGN.md §3 #14)
 *   the contributions to chunk c enter in rank order c, c+1, ..., c+P−1 (mod P)  (chunk (r−k) mod P
 *   is sent by rank r at reduce-scatter hop k)
 *     hop 0:   acc = s_c · g_c                  (fp32 multiply, then round to the storage dtype)
 *     hop h>0: acc = fmaf(s_r, g_r, acc)        (fp32 fused multiply-add, then round to the dtype)
 *   a rank with n_r = 0 contributes nothing (acc unchanged; 0 at hop 0).
 *
 * The fp64 weighted mean in wavg.py is the oracle proper; this emulation is the debugging aid that
 * a correct chunk/offset/order implementation matches bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static float bits_to_f32(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t f32_to_bits(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* round-to-nearest-even float32 -> bfloat16 (finite inputs; NaN -> quiet NaN) */
static uint16_t f32_to_bf16(float f) {
    uint32_t b = f32_to_bits(f);
    if (isnan(f)) return (uint16_t)((b >> 16) | 0x0040u);
    uint32_t lsb = (b >> 16) & 1u;
    return (uint16_t)((b + 0x7FFFu + lsb) >> 16);
}
static float bf16_to_f32(uint16_t h) { return bits_to_f32(((uint32_t)h) << 16); }

void ring_emulate_f32(int P, int64_t count, int64_t cs, const float *g /* [P][count] */,
                      const float *s /* [P] */, const int *active /* [P] */, float *out) {
    for (int c = 0; c < P; ++c) {
        int64_t lo = (int64_t)c * cs, hi = lo + cs;
        if (hi > count) hi = count;
        for (int64_t j = lo; j < hi; ++j) {
            float acc = 0.0f;
            for (int h = 0; h < P; ++h) {
                int r = (c + h) % P;
                if (!active[r]) continue;
                float x = g[(int64_t)r * count + j];
                if (h == 0) acc = s[r] * x;
                else acc = fmaf(s[r], x, acc);
            }
            out[j] = acc;
        }
    }
}

void ring_emulate_bf16(int P, int64_t count, int64_t cs, const uint16_t *g /* [P][count] bits */,
                       const float *s, const int *active, uint16_t *out) {
    for (int c = 0; c < P; ++c) {
        int64_t lo = (int64_t)c * cs, hi = lo + cs;
        if (hi > count) hi = count;
        for (int64_t j = lo; j < hi; ++j) {
            uint16_t acc = 0; /* +0.0 */
            for (int h = 0; h < P; ++h) {
                int r = (c + h) % P;
                if (!active[r]) continue;
                float x = bf16_to_f32(g[(int64_t)r * count + j]);
                if (h == 0) acc = f32_to_bf16(s[r] * x);
                else acc = f32_to_bf16(fmaf(s[r], x, bf16_to_f32(acc)));
            }
            out[j] = acc;
        }
    }
}
