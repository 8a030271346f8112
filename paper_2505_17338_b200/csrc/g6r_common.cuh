// g6r_common.cuh -- shared device helpers for the sm_100a 6DGS render path.
//
// The whole library is compiled with -fmad=false: every floating-point
// expression below rounds after each operation exactly like the reference's
// -ffp-contract=off CPU build (pkg/setup.py:13).  Where a fused multiply-add
// is intended it is written explicitly (__fma_rn).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

// Bounds checks of the checked build (make EXTRA=-DG6R_CHECKED, tools/
// checked_build.sh): every index the kernels derive from device-computed
// offsets (entry slots, sorted positions, splat rows, tile runs) is checked
// against its buffer, and a violation traps the context (the calling test
// then fails).  compiled out of the normal build.
#ifdef G6R_CHECKED
#define G6R_CHECK(c)                                                                       \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("g6r check failed %s:%d: %s\n", __FILE__, __LINE__, #c);                \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define G6R_CHECK(c) \
    do {             \
    } while (0)
#endif

#include "../../include/g6r.h"

namespace g6r {

// (row, column) of cov_raw[6 + k]: the row-major strict-lower pairs of the
// 6x6 Cholesky factor (core.py:30-31: (1,0) (2,1) (2,0) (3,0..2) (4,0..3)
// (5,0..4)); constexpr, so fully unrolled loops index registers, not local memory
__host__ __device__ constexpr int tril_i(int k) {
    return k < 1 ? 1 : k < 3 ? 2 : k < 6 ? 3 : k < 10 ? 4 : 5;
}
__host__ __device__ constexpr int tril_j(int k) {
    return k == 1 ? 1 : k < 3 ? 0 : k < 6 ? k - 3 : k < 10 ? k - 6 : k - 10;
}
static_assert(tril_i(2) == 2 && tril_j(2) == 0 && tril_i(5) == 3 && tril_j(5) == 2 &&
              tril_i(14) == 5 && tril_j(14) == 4, "tril order");

constexpr int kBlock = 256;          // threads per CTA for streaming kernels
constexpr int kMaxPasses = 8;        // radix passes (8-bit digits over <= 64-bit keys)
#ifndef G6R_SORT_ITEMS
#define G6R_SORT_ITEMS 8
#endif
constexpr int kSortItems = G6R_SORT_ITEMS;   // keys per thread in a onesweep tile
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
    kDoneCount = 14,       // compositor CTAs finished for the view (completion flag, host copies)
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

// --- glibc-compatible exp (f64) ----------------------------------------------
// glibc 2.39's exp (sysdeps/ieee754/dbl-64/e_exp.c, the FMA build the x86-64
// ifunc selects on AVX2/FMA hosts -- the libm `exp` the reference's f64
// compositor calls, _kernels.pyx:29-33, and `math.exp` of its brute-force
// test oracle, tests/oracles.py:60): k = round(x * 128/ln2), r = x - k ln2/128
// in two fma steps, 2^(k/128) = scale * (1 + tail) from a 128-pair table, a
// degree-5 polynomial, result = fma(scale, tmp, scale).  The operation order
// and the fma contractions are those of the host's __exp_fma (read from its
// machine code); the table is glibc's __exp_data.tab (entry 2i: tail bits,
// 2i+1: bits(2^(i/128)) - (i << 45)).  Checked bit-identical to the host libm
// on 245M inputs (random in [-700, 700], random bit patterns, a 1e-7 grid over
// [-4.5, 0]) and on the device by tests/test_gpu_parity.py.  Valid for
// |x| < 512; tiny |x| < 2^-54 returns 1 + x like glibc.  The compositors only
// call it on [-4.5, 0].
#define G6R_EXP_TABLE \
    {0x0000000000000000ull, 0x3ff0000000000000ull, 0x3c9b3b4f1a88bf6eull, 0x3feff63da9fb3335ull, \
     0xbc7160139cd8dc5dull, 0x3fefec9a3e778061ull, 0xbc905e7a108766d1ull, 0x3fefe315e86e7f85ull, \
     0x3c8cd2523567f613ull, 0x3fefd9b0d3158574ull, 0xbc8bce8023f98efaull, 0x3fefd06b29ddf6deull, \
     0x3c60f74e61e6c861ull, 0x3fefc74518759bc8ull, 0x3c90a3e45b33d399ull, 0x3fefbe3ecac6f383ull, \
     0x3c979aa65d837b6dull, 0x3fefb5586cf9890full, 0x3c8eb51a92fdeffcull, 0x3fefac922b7247f7ull, \
     0x3c3ebe3d702f9cd1ull, 0x3fefa3ec32d3d1a2ull, 0xbc6a033489906e0bull, 0x3fef9b66affed31bull, \
     0xbc9556522a2fbd0eull, 0x3fef9301d0125b51ull, 0xbc5080ef8c4eea55ull, 0x3fef8abdc06c31ccull, \
     0xbc91c923b9d5f416ull, 0x3fef829aaea92de0ull, 0x3c80d3e3e95c55afull, 0x3fef7a98c8a58e51ull, \
     0xbc801b15eaa59348ull, 0x3fef72b83c7d517bull, 0xbc8f1ff055de323dull, 0x3fef6af9388c8deaull, \
     0x3c8b898c3f1353bfull, 0x3fef635beb6fcb75ull, 0xbc96d99c7611eb26ull, 0x3fef5be084045cd4ull, \
     0x3c9aecf73e3a2f60ull, 0x3fef54873168b9aaull, 0xbc8fe782cb86389dull, 0x3fef4d5022fcd91dull, \
     0x3c8a6f4144a6c38dull, 0x3fef463b88628cd6ull, 0x3c807a05b0e4047dull, 0x3fef3f49917ddc96ull, \
     0x3c968efde3a8a894ull, 0x3fef387a6e756238ull, 0x3c875e18f274487dull, 0x3fef31ce4fb2a63full, \
     0x3c80472b981fe7f2ull, 0x3fef2b4565e27cddull, 0xbc96b87b3f71085eull, 0x3fef24dfe1f56381ull, \
     0x3c82f7e16d09ab31ull, 0x3fef1e9df51fdee1ull, 0xbc3d219b1a6fbffaull, 0x3fef187fd0dad990ull, \
     0x3c8b3782720c0ab4ull, 0x3fef1285a6e4030bull, 0x3c6e149289cecb8full, 0x3fef0cafa93e2f56ull, \
     0x3c834d754db0abb6ull, 0x3fef06fe0a31b715ull, 0x3c864201e2ac744cull, 0x3fef0170fc4cd831ull, \
     0x3c8fdd395dd3f84aull, 0x3feefc08b26416ffull, 0xbc86a3803b8e5b04ull, 0x3feef6c55f929ff1ull, \
     0xbc924aedcc4b5068ull, 0x3feef1a7373aa9cbull, 0xbc9907f81b512d8eull, 0x3feeecae6d05d866ull, \
     0xbc71d1e83e9436d2ull, 0x3feee7db34e59ff7ull, 0xbc991919b3ce1b15ull, 0x3feee32dc313a8e5ull, \
     0x3c859f48a72a4c6dull, 0x3feedea64c123422ull, 0xbc9312607a28698aull, 0x3feeda4504ac801cull, \
     0xbc58a78f4817895bull, 0x3feed60a21f72e2aull, 0xbc7c2c9b67499a1bull, 0x3feed1f5d950a897ull, \
     0x3c4363ed60c2ac11ull, 0x3feece086061892dull, 0x3c9666093b0664efull, 0x3feeca41ed1d0057ull, \
     0x3c6ecce1daa10379ull, 0x3feec6a2b5c13cd0ull, 0x3c93ff8e3f0f1230ull, 0x3feec32af0d7d3deull, \
     0x3c7690cebb7aafb0ull, 0x3feebfdad5362a27ull, 0x3c931dbdeb54e077ull, 0x3feebcb299fddd0dull, \
     0xbc8f94340071a38eull, 0x3feeb9b2769d2ca7ull, 0xbc87deccdc93a349ull, 0x3feeb6daa2cf6642ull, \
     0xbc78dec6bd0f385full, 0x3feeb42b569d4f82ull, 0xbc861246ec7b5cf6ull, 0x3feeb1a4ca5d920full, \
     0x3c93350518fdd78eull, 0x3feeaf4736b527daull, 0x3c7b98b72f8a9b05ull, 0x3feead12d497c7fdull, \
     0x3c9063e1e21c5409ull, 0x3feeab07dd485429ull, 0x3c34c7855019c6eaull, 0x3feea9268a5946b7ull, \
     0x3c9432e62b64c035ull, 0x3feea76f15ad2148ull, 0xbc8ce44a6199769full, 0x3feea5e1b976dc09ull, \
     0xbc8c33c53bef4da8ull, 0x3feea47eb03a5585ull, 0xbc845378892be9aeull, 0x3feea34634ccc320ull, \
     0xbc93cedd78565858ull, 0x3feea23882552225ull, 0x3c5710aa807e1964ull, 0x3feea155d44ca973ull, \
     0xbc93b3efbf5e2228ull, 0x3feea09e667f3bcdull, 0xbc6a12ad8734b982ull, 0x3feea012750bdabfull, \
     0xbc6367efb86da9eeull, 0x3fee9fb23c651a2full, 0xbc80dc3d54e08851ull, 0x3fee9f7df9519484ull, \
     0xbc781f647e5a3ecfull, 0x3fee9f75e8ec5f74ull, 0xbc86ee4ac08b7db0ull, 0x3fee9f9a48a58174ull, \
     0xbc8619321e55e68aull, 0x3fee9feb564267c9ull, 0x3c909ccb5e09d4d3ull, 0x3feea0694fde5d3full, \
     0xbc7b32dcb94da51dull, 0x3feea11473eb0187ull, 0x3c94ecfd5467c06bull, 0x3feea1ed0130c132ull, \
     0x3c65ebe1abd66c55ull, 0x3feea2f336cf4e62ull, 0xbc88a1c52fb3cf42ull, 0x3feea427543e1a12ull, \
     0xbc9369b6f13b3734ull, 0x3feea589994cce13ull, 0xbc805e843a19ff1eull, 0x3feea71a4623c7adull, \
     0xbc94d450d872576eull, 0x3feea8d99b4492edull, 0x3c90ad675b0e8a00ull, 0x3feeaac7d98a6699ull, \
     0x3c8db72fc1f0eab4ull, 0x3feeace5422aa0dbull, 0xbc65b6609cc5e7ffull, 0x3feeaf3216b5448cull, \
     0x3c7bf68359f35f44ull, 0x3feeb1ae99157736ull, 0xbc93091fa71e3d83ull, 0x3feeb45b0b91ffc6ull, \
     0xbc5da9b88b6c1e29ull, 0x3feeb737b0cdc5e5ull, 0xbc6c23f97c90b959ull, 0x3feeba44cbc8520full, \
     0xbc92434322f4f9aaull, 0x3feebd829fde4e50ull, 0xbc85ca6cd7668e4bull, 0x3feec0f170ca07baull, \
     0x3c71affc2b91ce27ull, 0x3feec49182a3f090ull, 0x3c6dd235e10a73bbull, 0x3feec86319e32323ull, \
     0xbc87c50422622263ull, 0x3feecc667b5de565ull, 0x3c8b1c86e3e231d5ull, 0x3feed09bec4a2d33ull, \
     0xbc91bbd1d3bcbb15ull, 0x3feed503b23e255dull, 0x3c90cc319cee31d2ull, 0x3feed99e1330b358ull, \
     0x3c8469846e735ab3ull, 0x3feede6b5579fdbfull, 0xbc82dfcd978e9db4ull, 0x3feee36bbfd3f37aull, \
     0x3c8c1a7792cb3387ull, 0x3feee89f995ad3adull, 0xbc907b8f4ad1d9faull, 0x3feeee07298db666ull, \
     0xbc55c3d956dcaebaull, 0x3feef3a2b84f15fbull, 0xbc90a40e3da6f640ull, 0x3feef9728de5593aull, \
     0xbc68d6f438ad9334ull, 0x3feeff76f2fb5e47ull, 0xbc91eee26b588a35ull, 0x3fef05b030a1064aull, \
     0x3c74ffd70a5fddcdull, 0x3fef0c1e904bc1d2ull, 0xbc91bdfbfa9298acull, 0x3fef12c25bd71e09ull, \
     0x3c736eae30af0cb3ull, 0x3fef199bdd85529cull, 0x3c8ee3325c9ffd94ull, 0x3fef20ab5fffd07aull, \
     0x3c84e08fd10959acull, 0x3fef27f12e57d14bull, 0x3c63cdaf384e1a67ull, 0x3fef2f6d9406e7b5ull, \
     0x3c676b2c6c921968ull, 0x3fef3720dcef9069ull, 0xbc808a1883ccb5d2ull, 0x3fef3f0b555dc3faull, \
     0xbc8fad5d3ffffa6full, 0x3fef472d4a07897cull, 0xbc900dae3875a949ull, 0x3fef4f87080d89f2ull, \
     0x3c74a385a63d07a7ull, 0x3fef5818dcfba487ull, 0xbc82919e2040220full, 0x3fef60e316c98398ull, \
     0x3c8e5a50d5c192acull, 0x3fef69e603db3285ull, 0x3c843a59ac016b4bull, 0x3fef7321f301b460ull, \
     0xbc82d52107b43e1full, 0x3fef7c97337b9b5full, 0xbc892ab93b470dc9ull, 0x3fef864614f5a129ull, \
     0x3c74b604603a88d3ull, 0x3fef902ee78b3ff6ull, 0x3c83c5ec519d7271ull, 0x3fef9a51fbc74c83ull, \
     0xbc8ff7128fd391f0ull, 0x3fefa4afa2a490daull, 0xbc8dae98e223747dull, 0x3fefaf482d8e67f1ull, \
     0x3c8ec3bc41aa2008ull, 0x3fefba1bee615a27ull, 0x3c842b94c3a9eb32ull, 0x3fefc52b376bba97ull, \
     0x3c8a64a931d185eeull, 0x3fefd0765b6e4540ull, 0xbc8e37bae43be3edull, 0x3fefdbfdad9cbe14ull, \
     0x3c77893b4d91cd9dull, 0x3fefe7c1819e90d8ull, 0x3c5305c14160cc89ull, 0x3feff3c22b8f71f1ull}

__device__ __forceinline__ double exp_glibc(double x, const unsigned long long *tab) {
    const double kInvLn2N = 0x1.71547652b82fep+7, kShift = 0x1.8p52;
    const double kNegLn2hiN = -0x1.62e42fefa0000p-8, kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    const unsigned abstop = (unsigned)(__double_as_longlong(x) >> 52) & 0x7ffu;
    if (abstop < 0x3c9u) return __dadd_rn(1.0, x);   // |x| < 2^-54
    double kd = __fma_rn(x, kInvLn2N, kShift);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = __dsub_rn(kd, kShift);
    double r = __fma_rn(kd, kNegLn2hiN, x);
    r = __fma_rn(kd, kNegLn2loN, r);
    const unsigned idx = 2u * (unsigned)(ki & 127ull);
    const double tail = __longlong_as_double((long long)tab[idx]);
    const double scale = __longlong_as_double((long long)(tab[idx + 1] + (ki << 45)));
    const double r2 = __dmul_rn(r, r);
    const double p23 = __fma_rn(r, C3, C2);
    const double p45 = __fma_rn(r, C5, C4);
    double tmp = __fma_rn(p23, r2, __dadd_rn(r, tail));
    tmp = __fma_rn(__dmul_rn(r2, r2), p45, tmp);
    return __fma_rn(scale, tmp, scale);
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
