// g6r_common.cuh -- shared device helpers for the sm_100a 6DGS render path.
//
// The whole library is compiled with -fmad=false: every floating-point
// expression below rounds after each operation exactly like the reference's
// -ffp-contract=off CPU build (pkg/setup.py:13).  Where a fused multiply-add
// is intended it is written explicitly (__fma_rn).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/g6r.h"

namespace g6r {

constexpr int kBlock = 256;          // threads per CTA for streaming kernels
constexpr int kMaxPasses = 8;        // radix passes (8-bit digits over <= 64-bit keys)
constexpr int kSortItems = 8;        // keys per thread in a onesweep tile
constexpr int kSortThreads = 256;    // threads per onesweep CTA
constexpr int kSortTile = kSortThreads * kSortItems;   // 2048 keys per tile
constexpr double kMinAlpha = 1.0 / 255.0;        // raster.py:47

constexpr int kRadixBits = 9;                    // LSD digit width
constexpr int kBins = 1 << kRadixBits;

// internal counter slots (int64) at the head of every workspace (zeroed per view)
enum {
    kTicketProject = 0,
    kTicketSortBase = 1,   // 1..8: one per radix pass
    kDepthMinInv = 10,     // ~min f32 depth bits of the drawn splats (atomicMax of ~bits)
    kDepthMax = 11,        // max f32 depth bits
    kValsBuffer = 9,       // which vals buffer holds the sorted entry values
    kSortPasses = 12,      // radix passes actually needed (decided on the device)
    kTicketComposite = 13, // compositor work-item ticket (slot of the batch's first view)
    kNumInternal = 16
};

// Which ping-pong buffer holds the sorted entry values after the radix passes.
__device__ __forceinline__ int sorted_buffer(const long long *internal) {
    return (int)(internal[kValsBuffer] & 1);
}

// Fold a CTA's depth-bit extrema (max of ~bits, max of bits) into the view's.
__device__ __forceinline__ void note_depth_extrema(long long *internal, unsigned lo_inv, unsigned hi) {
    atomicMax(reinterpret_cast<unsigned long long *>(&internal[kDepthMinInv]),
              (unsigned long long)lo_inv);
    atomicMax(reinterpret_cast<unsigned long long *>(&internal[kDepthMax]), (unsigned long long)hi);
}

// Per-splat compositing payload (f32): (mx, my, conic_a, conic_b),
// (conic_c, alpha, r, g), (b, cull_x, cull_y, -).  48 bytes, 16-byte aligned.
// cull_x/cull_y are conservative half-extents of the region where the
// compositor can see power >= -4.5 (see cull_extents); outside them every
// pixel skips the splat, so whole warps may skip it without changing a bit.
struct PayloadF32 {
    float4 a, b, c;
};
// f64 payload: 9 doubles + the two cull extents, 96 bytes (6 x double2).
struct PayloadF64 {
    double2 a, b, c, d, e;   // (mx,my) (ca,cb) (cc,alpha) (r,g) (b, cull_x)
    double2 f;               // (cull_y, -)
};

// Half-extents (px) of {q(dx,dy) = a dx^2 + 2 b dx dy + c dy^2 <= 9} -- the
// only pixels whose power = -q/2 can reach the [-4.5, 0] window -- inflated so
// the test stays conservative under the compositor's float rounding.  The
// computed q carries a relative error of at most ~10 ulp of
// (a dx^2 + c dy^2) <= 4 kappa q, kappa = (a+c)^2 / (4 det); outside the box
// grown by (1 + delta), delta >> 10 ulp * 4 kappa, the computed power is
// therefore still < -4.5.  Non-positive-definite conics get an infinite box.
// Squared-radius bound of the pixels a splat of peak alpha `alpha` can touch:
// a contribution needs power >= -4.5 (q <= 9) and alpha * exp(power) >= 1/255
// (q <= 2 ln(255 alpha)); the latter is tighter for alpha < e^4.5 / 255 (~0.35).
// Margins (1e-5 relative on alpha, 1e-4 absolute on q) cover the float
// rounding of expf and of the product in the compositor.  Returns a negative
// value when the splat can never pass the alpha floor.
__host__ __device__ __forceinline__ double cull_q(double alpha) {
    const double floor = 1.0 / 255.0;   // <= the f32 compositor's (float)(1/255)
    const double amax = alpha * (1.0 + 1e-5);
    if (!(amax > floor)) return -1.0;
    // single-precision log with generous margins (an upper bound is all we need)
    const double qa = 2.0 * (double)logf((float)(amax / floor)) * (1.0 + 1e-4) + 1e-3;
    return qa < 9.0 ? qa : 9.0;
}

__device__ __forceinline__ void cull_extents(double a, double b, double c, double ulp,
                                             float &ex, float &ey, double alpha = 1.0) {
    const double det = a * c - b * b;
    if (!(det > 0.0) || !(a > 0.0) || !(c > 0.0)) {
        ex = ey = __int_as_float(0x7f800000);
        return;
    }
    const double kappa = (a + c) * (a + c) / (4.0 * det);
    const double delta = 64.0 * ulp * kappa + 1e-6;
    if (!(delta < 0.5)) {
        ex = ey = __int_as_float(0x7f800000);
        return;
    }
    const double q = cull_q(alpha);
    if (q < 0.0) {   // can never reach the alpha floor: no pixel box at all
        ex = ey = __int_as_float(0x7fffffff);
        return;
    }
    const double grow = 1.0 + delta;
    const double k = sqrt(q);
    ex = (float)(k * sqrt(c / det) * grow + 1e-3);
    ey = (float)(k * sqrt(a / det) * grow + 1e-3);
}

// Same bound for the f32 compositor, in float with the SFU approximations
// (lg2, rcp, rsqrt; a few ulp each, far inside the 1e-4 / 1e-3 margins).  The
// compositor's alpha is al * expf(pw) <= al, so al < (float)(1/255) can never
// pass its floor; a NaN al would pass it wherever the power is in range.
__device__ __forceinline__ float cull_q_f32(float alpha) {
    const float floor_f = (float)(1.0 / 255.0);   // the compositor's floor_a
    if (alpha < floor_f) return -1.0f;
    if (!(alpha == alpha)) return 9.0f;
    // ln(alpha / floor_f) <= ln(255 alpha) since floor_f > 1/255
    const float qa = 2.0f * __logf(alpha * 255.0f) * (1.0f + 1e-4f) + 1e-3f;
    return qa < 9.0f ? qa : 9.0f;
}

// Lowest power at which a splat of peak alpha `alpha` can still pass the
// compositor's alpha floor: -q/2 for the (margined) cull_q bound, never below
// the -4.5 cutoff.  Below it alpha * expf(power) < 1/255 in the compositor's
// own rounding, so skipping those pixels before the expf changes no bit.
__device__ __forceinline__ float power_floor_f32(float alpha) {
    const float q = cull_q_f32(alpha);
    return q >= 0.0f ? fmaxf(-0.5f * q, -4.5f) : -4.5f;
}
__device__ __forceinline__ double power_floor(double alpha) {
    const double q = cull_q(alpha);
    return q >= 0.0 ? fmax(-0.5 * q, -4.5) : -4.5;
}

// Same extents for an f32 conic, in float arithmetic (the determinant exactly
// from the f32 products in double).  The float evaluation with approximate
// reciprocal / square roots adds at most a few ulp (~1e-6 relative); the
// extra 1e-5 relative growth absorbs it.
__device__ __forceinline__ void cull_extents_f32(float a, float b, float c, float &ex, float &ey,
                                                 float alpha = 1.0f) {
    const double detd = (double)a * (double)c - (double)b * (double)b;
    const float inf = __int_as_float(0x7f800000);
    if (!(detd > 0.0) || !(a > 0.0f) || !(c > 0.0f)) {
        ex = ey = inf;
        return;
    }
    const float inv = __fdividef(1.0f, (float)detd);
    const float kappa = (a + c) * (a + c) * 0.25f * inv;
    const float delta = 64.0f * 0x1p-23f * kappa + 1e-5f;
    if (!(delta < 0.5f)) {
        ex = ey = inf;
        return;
    }
    const float q = cull_q_f32(alpha);
    if (q < 0.0f) {
        ex = ey = __int_as_float(0x7fffffff);
        return;
    }
    const float grow = 1.0f + delta;
    const float k = q * rsqrtf(q) * (1.0f + 1e-6f);
    const float xc = c * inv, xa = a * inv;
    ex = k * (xc * rsqrtf(xc)) * grow + 1e-3f;
    ey = k * (xa * rsqrtf(xa)) * grow + 1e-3f;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Bit of the current device in a 64-bit per-device "done" mask (function
// attributes such as the dynamic shared-memory limit are per device/context).
inline unsigned long long device_bit() {
    int dev = 0;
    cudaGetDevice(&dev);
    return 1ull << (dev & 63);
}

// --- glibc-compatible expf --------------------------------------------------
// glibc 2.39 computes expf in double precision: k = round(x * 32/ln2),
// r = x*32/ln2 - k, 2^(k/32) from a 32-entry table, and a cubic in r
// (sysdeps/ieee754/flt-32/e_expf.c, FMA build selected on x86-64-v3 hosts).
// Reproducing that arithmetic exactly gives the reference's f32 compositor
// bits (raster.py:405-408 cast the splats to f32; _kernels.pyx:29-33 calls
// expf).  Verified against the host libm on all 2.24e9 floats in [-104, 88]
// (tests/test_expf_model.py runs the same model on the CPU).
// Table entries: bits(2^(i/32)) - (i << 47), i.e. the exponent field is
// re-added from k at run time.
#define G6R_EXPF_TABLE \
    {0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, \
     0x3fef9301d0125b51ull, 0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, \
     0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull, 0x3fef06fe0a31b715ull, \
     0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull, \
     0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, \
     0x3feea47eb03a5585ull, 0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, \
     0x3feea11473eb0187ull, 0x3feea589994cce13ull, 0x3feeace5422aa0dbull, \
     0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull, \
     0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, \
     0x3fef3720dcef9069ull, 0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, \
     0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull}

__device__ __forceinline__ float expf_glibc(float x, const unsigned long long *tab) {
    const double kInvLn2N = 0x1.71547652b82fep+5;   // 32 / ln 2
    const double kShift = 0x1.8p+52;
    const double c0 = 0x1.c6af84b912394p-20;         // poly scaled by 32^-3
    const double c1 = 0x1.ebfce50fac4f3p-13;         // 32^-2
    const double c2 = 0x1.62e42ff0c52d6p-6;          // 32^-1
    const double xd = (double)x;
    const double z = __dmul_rn(kInvLn2N, xd);
    double kd = __dadd_rn(z, kShift);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = __dsub_rn(kd, kShift);
    const double r = __fma_rn(kInvLn2N, xd, -kd);
    const unsigned long long t = tab[ki & 31ull] + (ki << 47);
    const double s = __longlong_as_double((long long)t);
    const double p = __fma_rn(c0, r, c1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(c2, r, 1.0);
    y = __fma_rn(p, r2, y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

// x86 cvttsd2si semantics for the radius cast (_kernels.pyx:346): NaN -> INT_MIN.
__device__ __forceinline__ int32_t cast_i32_x86(double v) {
    if (isnan(v)) return INT32_MIN;
    return (int32_t)v;
}

// --- small block-scan helpers ---------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// GPU-scope relaxed accesses for look-back status words (volatile compiles to
// system-scope strong accesses, which the look-back does not need).
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned *p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u32(unsigned *p, unsigned v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace g6r
