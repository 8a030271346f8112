// g6r_composite.cu -- per-tile front-to-back alpha compositing (forward) and
// its adjoint.
//
// Replaces raster.py:392-415 _composite -> _kernels.pyx:36-105
// composite_forward (and :108-187 composite_backward).  One CTA per screen
// tile, one thread per pixel.  Each CTA walks its depth-sorted run in batches
// of blockDim splats: the batch's payloads are gathered once into shared
// memory (every pixel then reads them as broadcasts) and the CTA stops as soon
// as __syncthreads_count reports every pixel saturated (T < 1e-4).  Pixel
// arithmetic is the reference's f32 expression order with no contraction, and
// expf is evaluated with glibc's algorithm (g6r_common.cuh), so the f32
// framebuffer matches the reference's bit for bit.  Nothing here is a dense
// contraction, so it runs on the FP32/FP64 pipes, not tensor cores.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <atomic>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

#ifndef G6R_GROUPED_MINB
#define G6R_GROUPED_MINB 8   // min CTAs/SM for the grouped f32 compositor (<= 64 registers)
#endif
#ifndef G6R_SCHED_MINB
#define G6R_SCHED_MINB 0   // min CTAs/SM for the scheduled f32 compositor (A/B knob)
#endif

__constant__ unsigned long long c_expf_tab[32] = G6R_EXPF_TABLE;
__constant__ unsigned long long c_exp_tab[256] = G6R_EXP_TABLE;   // f64 glibc exp

template <typename Real>
struct Px;

// Shared-memory splat record: two 16-byte vectors + the blue channel, so the
// per-hit reads are LDS.128 x2 (+1) instead of nine scalar loads.
template <>
struct Px<float> {
    using Payload = PayloadF32;
    struct alignas(16) S {
        float4 a;   // mx, my, conic a, conic b
        float4 b;   // conic c, alpha, r, g
        float2 c;   // b, power floor
    };
    __device__ static S unpack(const Payload &p, float &ex, float &ey) {
        ex = p.c.y;
        ey = p.c.z;
        S s;
        s.a = p.a;
        s.b = p.b;
        s.c = make_float2(p.c.x, p.c.w);
        return s;
    }
    __device__ static float mx(const S &s) { return s.a.x; }
    __device__ static float my(const S &s) { return s.a.y; }
};
template <>
struct Px<double> {
    using Payload = PayloadF64;
    struct alignas(16) S {
        double2 a, b, c, d;   // (mx,my) (ca,cb) (cc,alpha) (r,g)
        double2 e;            // (b, power floor)
    };
    __device__ static S unpack(const Payload &p, float &ex, float &ey) {
        ex = (float)p.e.y;
        ey = (float)p.f.x;
        S s;
        s.a = p.a;
        s.b = p.b;
        s.c = p.c;
        s.d = p.d;
        s.e = make_double2(p.e.x, p.f.y);
        return s;
    }
    __device__ static double mx(const S &s) { return s.a.x; }
    __device__ static double my(const S &s) { return s.a.y; }
};

// Field access common to both layouts.
__device__ __forceinline__ void fields(const Px<float>::S &s, float &mx, float &my, float &ca,
                                       float &cb, float &cc, float &al) {
    mx = s.a.x; my = s.a.y; ca = s.a.z; cb = s.a.w; cc = s.b.x; al = s.b.y;
}
__device__ __forceinline__ void colours(const Px<float>::S &s, float &r, float &g, float &b) {
    r = s.b.z; g = s.b.w; b = s.c.x;
}
__device__ __forceinline__ float power_lo(const Px<float>::S &s) { return s.c.y; }
__device__ __forceinline__ void fields(const Px<double>::S &s, double &mx, double &my, double &ca,
                                       double &cb, double &cc, double &al) {
    mx = s.a.x; my = s.a.y; ca = s.b.x; cb = s.b.y; cc = s.c.x; al = s.c.y;
}
__device__ __forceinline__ void colours(const Px<double>::S &s, double &r, double &g, double &b) {
    r = s.d.x; g = s.d.y; b = s.e.x;
}
__device__ __forceinline__ double power_lo(const Px<double>::S &s) { return s.e.y; }

// Pixel of thread t in a tile: 16x16 tiles give each warp an 8x4 block (so the
// per-warp culling box is square-ish); other tile sizes are row-major.
__device__ __forceinline__ void tile_pixel(int ts, int t, int &dx, int &dy) {
    if (ts == 16) {
        const int w = t >> 5, l = t & 31;
        dx = (w & 1) * 8 + (l & 7);
        dy = (w >> 1) * 4 + (l >> 3);
    } else {
        dx = t % ts;
        dy = t / ts;
    }
}

// Grouped hit lists (16x16 tiles split into 16x8 bands, 4 warps of 8x4):
// the warp's 32 lanes form kG groups of gw x gh pixels, each walking its own
// hit list, so a small splat costs one pass of the group(s) it can touch
// rather than of the whole warp.  Lane l of warp w: group g = l / (32/kG),
// pixel (bx + group origin + lane-in-group offset).
template <int kG> struct GroupShape;
template <> struct GroupShape<1> { static constexpr int w = 8, h = 4; };
template <> struct GroupShape<2> { static constexpr int w = 4, h = 4; };
template <> struct GroupShape<4> { static constexpr int w = 4, h = 2; };
template <> struct GroupShape<8> { static constexpr int w = 2, h = 2; };

// 32x32 bit-matrix transpose across a warp: in, lane i bit b; out, lane b
// bit i (five butterfly stages, each swapping the off-diagonal blocks).
template <int J, unsigned M0>
__device__ __forceinline__ unsigned transpose_stage(unsigned x, int lane) {
    const unsigned y = __shfl_xor_sync(0xffffffffu, x, J);
    const unsigned hi = (x & ~M0) | ((y & ~M0) >> J);   // lanes with bit J set
    const unsigned lo = (x & M0) | ((y & M0) << J);
    return (lane & J) ? hi : lo;
}
__device__ __forceinline__ unsigned warp_transpose32(unsigned x, int lane) {
    x = transpose_stage<16, 0x0000ffffu>(x, lane);
    x = transpose_stage<8, 0x00ff00ffu>(x, lane);
    x = transpose_stage<4, 0x0f0f0f0fu>(x, lane);
    x = transpose_stage<2, 0x33333333u>(x, lane);
    return transpose_stage<1, 0x55555555u>(x, lane);
}

template <int kG>
__device__ __forceinline__ void band_pixel(int t, int &dx, int &dy) {
    constexpr int gw = GroupShape<kG>::w, gh = GroupShape<kG>::h, gpr = 8 / gw;
    const int w = t >> 5, l = t & 31;
    const int g = l / (32 / kG), i = l % (32 / kG);
    dx = (w & 1) * 8 + (g % gpr) * gw + i % gw;
    dy = (w >> 1) * 4 + (g / gpr) * gh + i / gw;
}
// bit of the band's sub-block grid (16/gw columns x 8/gh rows, row-major)
// holding band pixel (dx, dy)
template <int kG>
__device__ __forceinline__ int group_bit(int dx, int dy) {
    constexpr int gw = GroupShape<kG>::w, gh = GroupShape<kG>::h;
    return (dy / gh) * (16 / gw) + dx / gw;
}

__device__ __forceinline__ float splat_exp(float x, const unsigned long long *tab) {
    return expf_glibc(x, tab);
}
__device__ __forceinline__ double splat_exp(double x, const unsigned long long *) { return exp(x); }

// Shared-memory reads through 32-bit shared-window addresses held in
// registers: generic pointers into shared memory make the compiler rebuild the
// window base (S2R CgaCtaId + LEA) at every use inside the hit loop.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void lds_splat(uint32_t a, Px<float>::S &s) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(s.a.x), "=f"(s.a.y), "=f"(s.a.z), "=f"(s.a.w) : "r"(a));
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+16];"
                 : "=f"(s.b.x), "=f"(s.b.y), "=f"(s.b.z), "=f"(s.b.w) : "r"(a));
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2+32];" : "=f"(s.c.x), "=f"(s.c.y) : "r"(a));
}
__device__ __forceinline__ void lds_splat(uint32_t a, Px<double>::S &s) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(s.a.x), "=d"(s.a.y) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+16];" : "=d"(s.b.x), "=d"(s.b.y) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+32];" : "=d"(s.c.x), "=d"(s.c.y) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+48];" : "=d"(s.d.x), "=d"(s.d.y) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+64];" : "=d"(s.e.x), "=d"(s.e.y) : "r"(a));
}
__device__ __forceinline__ unsigned lds_u32(uint32_t a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned long long lds_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}

// Operands of the hit loop's expf.  The 64-bit constants live in the constant
// bank, which DMUL/DFMA read directly (c[bank][offset] operands); as literals
// ptxas rebuilds them with 32-bit moves on every splat visit.  The table's
// window address goes through an opaque move for the same reason.
__constant__ double c_exp_k[4] = {0x1.71547652b82fep+5, 0x1.c6af84b912394p-20,
                                  0x1.ebfce50fac4f3p-13, 0x1.62e42ff0c52d6p-6};
struct ExpOperands {
    uint32_t tab;
};
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ ExpOperands exp_operands(uint32_t tab) { return ExpOperands{opaque(tab)}; }
__device__ __forceinline__ uint2 lds_u32x2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// glibc expf (g6r_common.cuh expf_glibc, same operations) with the operands
// above.  The scale 2^(k/32) is the table entry with k's low 17 bits added to
// its exponent field: (k << 47) only touches the high word, so one 32-bit add.
__device__ __forceinline__ float splat_exp_s(float x, const ExpOperands &e) {
    const double kInvLn2N = c_exp_k[0];
    const double kShift = 0x1.8p+52;
    const double c0 = c_exp_k[1], c1 = c_exp_k[2], c2 = c_exp_k[3];
    const uint32_t tab = e.tab;
    const double xd = (double)x;
    const double z = __dmul_rn(kInvLn2N, xd);
    double kd = __dadd_rn(z, kShift);
    const unsigned ki = (unsigned)__double2loint(kd);
    kd = __dsub_rn(kd, kShift);
    const double r = __fma_rn(kInvLn2N, xd, -kd);
    const uint2 t = lds_u32x2(tab + 8u * (ki & 31u));
    const double s = __hiloint2double((int)(t.y + (ki << 15)), (int)t.x);
    const double p = __fma_rn(c0, r, c1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(c2, r, 1.0);
    y = __fma_rn(p, r2, y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}
__device__ __forceinline__ double splat_exp_s(double x, const ExpOperands &) { return exp(x); }

// View completion (g6r_frame.host_image / host_rgba8): every CTA of a view,
// after its pixels are stored, bumps the view's CTA counter (gpu-scope fence
// first); the last one publishes done_value to the view's flag with a
// system-scope release, which gates the host copy enqueued on the copy stream
// (cuStreamWaitValue32, g6r_api.cu).
__device__ __forceinline__ void signal_view_done(const Batch &bt, int view, int sub) {
    __syncthreads();
    const ViewOut &o = bt.out[view];
    if (threadIdx.x != 0 || !o.done_flag) return;
    __threadfence();
    const unsigned long long total =
        (unsigned long long)bt.vp[view].tiles_x * bt.vp[view].tiles_y * (unsigned long long)sub;
    const unsigned long long prev =
        atomicAdd(reinterpret_cast<unsigned long long *>(&bt.ws[view].internal[kDoneCount]), 1ull);
    if (prev + 1 == total) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(o.done_flag), "r"(o.done_value) : "memory");
    }
}

#ifdef G6R_CTA_TRACE
// Debug build only (-DG6R_CTA_TRACE): per compositor CTA (globaltimer start,
// end, SM, view << 16 | item, run length), read by g6r_debug_cta_trace.
__device__ unsigned long long g_cta_trace[1 << 17][4];
__device__ unsigned g_cta_trace_n;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

// One CTA per tile, one thread per pixel.  kNB > 0: compile-time block size
// (16x16 tiles, static shared memory); kNB == 0: any tile size up to 32x32.
//
// The run is consumed in batches of blockDim entries, double-buffered: the
// gather of batch k+1 (payload[vals[e]], L2-resident) is issued into registers
// before batch k is composited and lands in the other shared buffer after, so
// its latency hides behind compute and each batch costs one barrier.  The
// staging thread also tests the splat's conservative 3-sigma box against every
// warp's pixel block; warps then ballot over the batch and visit only splats
// that can touch them, in ascending order (the per-pixel order, hence every
// bit, is unchanged).
template <typename Real, int kNB, int kSub = 1, bool kFastExp = false, bool kSched = false, int kG = 1>
__global__ void __launch_bounds__(kNB > 0 ? kNB : 1024,
                                  (kG > 1 && sizeof(Real) == 4) ? G6R_GROUPED_MINB
                                  : (kSched && sizeof(Real) == 4) ? G6R_SCHED_MINB : 0)
k_composite(const __grid_constant__ Batch bt, int sorted) {
    constexpr bool scheduled = kSched && kSub > 1;
    constexpr bool grouped = kG > 1 && kNB == 128 && kSub == 2;
    using S = typename Px<Real>::S;
    // Work item: with `scheduled` (kSub > 1), CTAs take (view, tile) items in
    // k_sched_order's longest-run-first order through a ticket, both bands of
    // a tile back to back, so the batch's heaviest runs start first and the
    // launch's tail is made of short ones; otherwise blockIdx names the item.
    __shared__ unsigned s_item;
    if (kSub > 1 && scheduled) {
        if (threadIdx.x == 0) {
            const unsigned k = (unsigned)atomicAdd(
                reinterpret_cast<unsigned long long *>(&bt.ws[0].internal[kTicketComposite]), 1ull);
            const int T = bt.vp[0].tiles_x * bt.vp[0].tiles_y;
            const unsigned r = k / kSub;
            const unsigned it = bt.ws[r / T].sched[r % T];
            s_item = ((it >> 16) << 16) | ((it & 0xffffu) * kSub + k % kSub);
        }
        __syncthreads();
    }
    // This thread's (view, pixel).  Derived from blockIdx or from the shared
    // work item, and derived again in the epilogue instead of being kept: the
    // view index and pixel coordinates then hold no registers across the
    // compositing loop (with the scheduled item they could not be
    // rematerialised from special registers).
    struct Where {
        int view, tile, band, px, py;
        bool inside;
    };
    auto where = [&]() {
        Where w;
        int item_x;
        if (kSub > 1 && scheduled) {
            unsigned it;
            asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(it) : "r"(smem_addr(&s_item)));
            w.view = (int)(it >> 16);
            item_x = (int)(it & 0xffffu);
        } else {
            w.view = blockIdx.y;
            item_x = blockIdx.x;
        }
        const ViewParams &v = bt.vp[w.view];
        const int ts_ = v.tile_size;
        // kSub > 1 (16x16 tiles only): the tile's rows are split over kSub
        // CTAs, each walking the whole run for its band, so a band that
        // saturates early frees its SM slot instead of idling at the other
        // band's barriers
        w.tile = kSub > 1 ? item_x / kSub : item_x;
        w.band = kSub > 1 ? (item_x % kSub) * (16 / kSub) : 0;
        int ox, oy;
        if constexpr (grouped)
            band_pixel<kG>(threadIdx.x, ox, oy);
        else
            tile_pixel(ts_, threadIdx.x, ox, oy);
        w.px = (w.tile % v.tiles_x) * ts_ + ox;
        w.py = (w.tile / v.tiles_x) * ts_ + oy + w.band;
        w.inside = w.px < v.iw && w.py < v.ih;
        return w;
    };
#ifdef G6R_CTA_TRACE
    const unsigned long long t_start = gtimer();
#endif
    const Where at = where();
    const int view = at.view;
    const ViewParams &vp = bt.vp[view];
    const Workspace &wsv = bt.ws[view];
    const typename Px<Real>::Payload *__restrict__ payload =
        static_cast<const typename Px<Real>::Payload *>(wsv.payload);
    const int64_t *__restrict__ starts = wsv.tile_starts;
    constexpr int kStatic = kNB > 0 ? kNB : 1;
    __shared__ S s_sp_static[kNB > 0 ? 2 * kStatic : 1];
    __shared__ unsigned s_mask_static[kNB > 0 ? 2 * kStatic : 1];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nb = kNB > 0 ? kNB : (int)blockDim.x;
    S *sp = kNB > 0 ? s_sp_static : reinterpret_cast<S *>(smem_raw);
    unsigned *smask = kNB > 0 ? s_mask_static : reinterpret_cast<unsigned *>(sp + 2 * nb);
    __shared__ unsigned long long s_tab[32];
    __shared__ unsigned long long s_tab64[sizeof(Real) == 8 ? 256 : 1];
    __shared__ float4 s_wbox[32];   // pixel-centre box per warp
    for (int k = threadIdx.x; k < 32; k += blockDim.x) s_tab[k] = c_expf_tab[k];   // tiles below 6x6 have < 32 threads
    if constexpr (sizeof(Real) == 8)
        for (int k = threadIdx.x; k < 256; k += blockDim.x) s_tab64[k] = c_exp_tab[k];
    const uint32_t sp_base = smem_addr(sp), mask_base = smem_addr(smask);
    const ExpOperands eops = exp_operands(smem_addr(s_tab));

    const int ts = vp.tile_size;
    const int tile = at.tile, band = at.band;
    const int tx = tile % vp.tiles_x, ty = tile / vp.tiles_x;
    const bool inside = at.inside;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = (nb + 31) >> 5;
    const int wlanes = min(32, nb - warp * 32);
    const unsigned wmask = wlanes == 32 ? 0xffffffffu : ((1u << wlanes) - 1u);
    if (threadIdx.x < nwarps) {   // pixel-centre box of warp w, clipped to the image
        const int w = threadIdx.x;
        int x0, x1, y0, y1;
        if (ts == 16) {
            x0 = (w & 1) * 8;
            x1 = x0 + 7;
            y0 = (w >> 1) * 4 + band;
            y1 = y0 + 3;
        } else {
            const int t0 = w * 32, t1 = min(nb, t0 + 32) - 1;
            y0 = t0 / ts;
            y1 = t1 / ts;
            x0 = y0 == y1 ? t0 % ts : 0;
            x1 = y0 == y1 ? t1 % ts : ts - 1;
        }
        x0 += tx * ts;
        x1 = min(x1 + tx * ts, vp.iw - 1);
        y0 += ty * ts;
        y1 = min(y1 + ty * ts, vp.ih - 1);
        s_wbox[w] = (x0 <= x1 && y0 <= y1) ? make_float4((float)x0, (float)x1, (float)y0, (float)y1)
                                           : make_float4(1e30f, -1e30f, 1e30f, -1e30f);
    }
    // the gather's two base pointers live in shared memory and are re-read per
    // batch (4 registers fewer across the compositing loop)
    __shared__ __align__(16) const void *s_gather[2];
    if (threadIdx.x == 0) {
        s_gather[0] = payload;
        s_gather[1] = wsv.vals[sorted ? sorted_buffer(wsv.internal) : 0];
    }
    auto gather = [&](int64_t e) {
        const void *pl, *vl;
        asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                     : "=l"(pl), "=l"(vl) : "r"(smem_addr(s_gather)));
        const unsigned idx = __ldg(static_cast<const unsigned *>(vl) + e);
        G6R_CHECK((int64_t)idx < bt.ws[view].nrows);
        return static_cast<const typename Px<Real>::Payload *>(pl)[idx];
    };
    const int64_t lo = starts[tile], hi = starts[tile + 1];
    G6R_CHECK(0 <= lo && lo <= hi && (wsv.entry_capacity <= 0 || hi <= wsv.entry_capacity));
    const Real fx = (Real)at.px, fy = (Real)at.py;
    const Real floor_a = (Real)(1.0 / 255.0), t_stop = (Real)1e-4;
    const Real half = (Real)-0.5, one = (Real)1;
    // a pixel is finished once T < t_stop (T never grows); pixels outside the
    // image start finished
    Real T = inside ? one : (Real)0, ar = 0, ag = 0, ab = 0, aa = 0;
    int last = 0;
    // fast exp: within 2.5e-6 (> 2e-6 + the ex2 error) of the alpha floor the
    // exact expf decides, so every floor decision is the exact mode's
    const float floor_lo = (float)(1.0 / 255.0) * (1.0f - 2.5e-6f);
    const float floor_hi = (float)(1.0 / 255.0) * (1.0f + 2.5e-6f);
    __syncthreads();   // s_wbox / s_tab ready

    // grouped: the band's pixel origin and last pixel inside the image
    const int gx0 = tx * ts, gy0 = ty * ts + band;
    const int gxmax = min(15, vp.iw - 1 - gx0), gymax = min(7, vp.ih - 1 - gy0);
    // grouped staging: the entry's box as a mask over the band's 32 sub-blocks
    // (16/gw columns x 8/gh rows), then the warp's 32 masks (one chunk of 32
    // entries) transposed so that lane b holds sub-block b's hit word for the
    // chunk: the hit loop reads its group's word with one shared load
    auto stage_grouped = [&](int buf, const typename Px<Real>::Payload &pl, bool have) {
        unsigned m = 0;
        if (have) {
            float ex, ey;
            const S s = Px<Real>::unpack(pl, ex, ey);
            sp[buf * nb + threadIdx.x] = s;
            const float mx = (float)Px<Real>::mx(s), my = (float)Px<Real>::my(s);
            // pixel columns/rows the box can touch: x >= fl(mx - ex) and
            // x <= fl(mx + ex), the same float tests as the per-warp box
            constexpr int gw = GroupShape<kG>::w, gh = GroupShape<kG>::h, ncol = 16 / gw;
            const int xl = max(__float2int_ru(mx - ex) - gx0, 0);
            const int xh = min(__float2int_rd(mx + ex) - gx0, gxmax);
            const int yl = max(__float2int_ru(my - ey) - gy0, 0);
            const int yh = min(__float2int_rd(my + ey) - gy0, gymax);
            if (xl <= xh && yl <= yh) {
                const unsigned cols = (2u << (xh / gw)) - (1u << (xl / gw));
#pragma unroll
                for (int r = 0; r < 8 / gh; ++r)
                    if (r >= yl / gh && r <= yh / gh) m |= cols << (r * ncol);
            }
        }
        smask[buf * nb + threadIdx.x] = warp_transpose32(m, lane);
    };
    // stage batch k's entry (this thread's) into buffer `buf`
    auto stage = [&](int64_t b0, int buf, const typename Px<Real>::Payload &pl, bool have) {
        if constexpr (grouped) {   // warp-collective (the transpose below)
            stage_grouped(buf, pl, have);
            return;
        }
        if (!have) return;
        float ex, ey;
        const S s = Px<Real>::unpack(pl, ex, ey);
        sp[buf * nb + threadIdx.x] = s;
        const float mx = (float)Px<Real>::mx(s), my = (float)Px<Real>::my(s);
        unsigned m = 0;
        {
            for (int w = 0; w < nwarps; ++w) {
                const float4 bx = s_wbox[w];
                if (mx + ex >= bx.x && mx - ex <= bx.y && my + ey >= bx.z && my - ey <= bx.w) m |= 1u << w;
            }
        }
        smask[buf * nb + threadIdx.x] = m;
    };
    // grouped: this lane's sub-block (its group's hit word in each chunk)
    int mybit = 0;
    if constexpr (grouped) {
        int ox, oy;
        band_pixel<kG>(threadIdx.x, ox, oy);
        mybit = group_bit<kG>(ox, oy);
    }

    typename Px<Real>::Payload pre;
    bool have = lo + threadIdx.x < hi;
    if (have) pre = gather(lo + threadIdx.x);
    stage(lo, 0, pre, have);
    __syncthreads();
    int buf = 0;
    for (int64_t b0 = lo; b0 < hi; b0 += nb, buf ^= 1) {
        // issue the next batch's gather now; it lands while this batch composites
        const int64_t e1 = b0 + nb + threadIdx.x;
        const bool have1 = e1 < hi;
        if (have1) pre = gather(e1);
        const uint32_t bsp = sp_base + (uint32_t)(buf * nb) * (uint32_t)sizeof(S);
        const uint32_t bmask = mask_base + (uint32_t)(buf * nb) * 4u;
        const int cnt = (int)((hi - b0) < nb ? (hi - b0) : nb);
        const int jbase = (int)(b0 - lo) + 1;   // last_contrib of batch entry j = jbase + j
        if (!__all_sync(wmask, T < t_stop)) {
            for (int c0 = 0; c0 < cnt; c0 += 32) {
                unsigned hits = 0;   // splats c0..c0+31 that can touch this warp (group)
                if constexpr (grouped) {
                    hits = lds_u32(bmask + 4u * (uint32_t)(c0 + mybit));
                } else {
                    for (int k = 0; k < 32; k += wlanes) {
                        const int jl = c0 + k + lane;
                        const unsigned b = __ballot_sync(
                            wmask, lane + k < 32 && jl < cnt && ((lds_u32(bmask + 4u * jl) >> warp) & 1u));
                        hits |= b << k;
                    }
                }
                // ascending order: walk the bit-reversed mask from its top bit;
                // grouped: the warp iterates as often as its busiest group
                unsigned rh = __brev(hits);
                if constexpr (grouped) {
                    // Branch-free visits: every lane runs the whole visit and
                    // a lane with nothing to add (its group's list exhausted,
                    // pixel finished, power out of range, below the alpha
                    // floor) adds exactly nothing (ai = 0: r*0 = 0, ar + 0 = ar,
                    // T*1 = T) -- the warp executes the union of the paths
                    // anyway, so the branches only cost divergence bookkeeping.
                    for (int it = __reduce_max_sync(0xffffffffu, (unsigned)__popc(hits)); it > 0; --it) {
                        const bool live = rh != 0u;
                        unsigned k;   // leading zeros of rh (FLO.SH; ~0 when rh == 0)
                        asm("bfind.shiftamt.u32 %0, %1;" : "=r"(k) : "r"(rh));
                        k = live ? k : 0u;
                        rh &= ~(0x80000000u >> k);
                        const int j = c0 + (int)k;
                        S s;
                        lds_splat(bsp + (uint32_t)j * (uint32_t)sizeof(S), s);
                        Real mx, my, ca, cb, cc, al;
                        fields(s, mx, my, ca, cb, cc, al);
                        const Real dx = fx - mx;
                        const Real dy = fy - my;
                        const Real pw = half * (ca * dx * dx + cc * dy * dy) - cb * dx * dy;
                        bool ok = live && !(T < t_stop) && !(pw > (Real)0) && !(pw < power_lo(s));
                        Real ai;
                        if constexpr (kFastExp) {
                            float e;
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(pw * 1.44269504088896341f));
                            ai = al * e;
                            if (ok && ai < floor_hi && ai >= floor_lo) ai = al * splat_exp_s(pw, eops);
                        } else if constexpr (sizeof(Real) == 8) {
                            ai = al * exp_glibc(pw, s_tab64);   // libm exp, bit for bit
                        } else {
                            ai = al * splat_exp_s(pw, eops);
                        }
                        ok = ok && !(ai < floor_a);
                        ai = ok ? ai : (Real)0;
                        Real r, g, b;
                        colours(s, r, g, b);
                        const Real w = ai * T;
                        if constexpr (kFastExp) {
                            ar = __fmaf_rn(r, w, ar);
                            ag = __fmaf_rn(g, w, ag);
                            ab = __fmaf_rn(b, w, ab);
                        } else {
                            ar = ar + r * w;
                            ag = ag + g * w;
                            ab = ab + b * w;
                        }
                        aa = aa + w;
                        T = T * (one - ai);
                        last = ok ? jbase + j : last;
                    }
                    continue;
                }
                while (rh != 0u) {
                    unsigned k;   // leading zeros of rh (FLO.SH)
                    asm("bfind.shiftamt.u32 %0, %1;" : "=r"(k) : "r"(rh));
                    rh ^= 0x80000000u >> k;
                    const int j = c0 + (int)k;
                    if (T < t_stop) continue;   // the pixel is finished
                    S s;
                    lds_splat(bsp + (uint32_t)j * (uint32_t)sizeof(S), s);
                    Real mx, my, ca, cb, cc, al;
                    fields(s, mx, my, ca, cb, cc, al);
                    const Real dx = fx - mx;
                    const Real dy = fy - my;
                    const Real pw = half * (ca * dx * dx + cc * dy * dy) - cb * dx * dy;
                    // power_lo >= -4.5: below it the alpha floor rejects the
                    // pixel anyway, so the expf is skipped, no bit changes
                    if (pw > (Real)0 || pw < power_lo(s)) continue;
                    Real ai;
                    if constexpr (kFastExp && sizeof(Real) == 4) {
                        // SFU 2^x: <= ~7e-7 relative from the exact path (ex2
                        // 2 ulp + the rounding of pw * log2 e for |pw| <= 4.5);
                        // inside 2e-6 of the floor the exact expf decides
                        float e;
                        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(pw * 1.44269504088896341f));
                        ai = al * e;
                        // one compare in the common case (well above the floor)
                        if (ai < floor_hi) {
                            if (ai >= floor_lo) ai = al * splat_exp_s(pw, eops);
                            if (ai < floor_a) continue;
                        }
                    } else {
                        if constexpr (sizeof(Real) == 8)
                            ai = al * exp_glibc(pw, s_tab64);   // libm exp, bit for bit
                        else
                            ai = al * splat_exp_s(pw, eops);
                        if (ai < floor_a) continue;
                    }
                    Real r, g, b;
                    colours(s, r, g, b);
                    const Real w = ai * T;
                    if constexpr (kFastExp && sizeof(Real) == 4) {
                        // fast mode: fused accumulation (one rounding per
                        // channel instead of two; T, and with it every
                        // termination decision, is computed as in exact mode)
                        ar = __fmaf_rn(r, w, ar);
                        ag = __fmaf_rn(g, w, ag);
                        ab = __fmaf_rn(b, w, ab);
                    } else {
                        ar = ar + r * w;
                        ag = ag + g * w;
                        ab = ab + b * w;
                    }
                    aa = aa + w;
                    T = T * (one - ai);
                    last = jbase + j;
                }
            }
        }
        // the other buffer was last read in the previous batch (fenced by the
        // barrier that ended it), so the prefetched splat can land there now
        stage(b0 + nb, buf ^ 1, pre, have1);
        if (__syncthreads_count(!(T < t_stop)) == 0) break;
    }
    const Where fin = where();
    if (fin.inside) {
        const ViewOut &out = bt.out[fin.view];
        Real *__restrict__ image = static_cast<Real *>(out.image);
        Real *__restrict__ final_t = static_cast<Real *>(out.final_t);
        int32_t *__restrict__ last_contrib = out.last_contrib;
        const int64_t p = (int64_t)fin.py * bt.vp[fin.view].iw + fin.px;
        if (image) {
            if constexpr (sizeof(Real) == 4) {
                reinterpret_cast<float4 *>(image)[p] = make_float4(ar, ag, ab, aa);
            } else {
                reinterpret_cast<double2 *>(image)[2 * p] = make_double2(ar, ag);
                reinterpret_cast<double2 *>(image)[2 * p + 1] = make_double2(ab, aa);
            }
        }
        if (uint8_t *q = out.rgba8) {
            // composite_over (metrics.py:24) then to_rgba_u8 (_png.py:30), in f64
            const double *bg = out.bg;
            const double t = 1.0 - (double)aa;
            const double c[3] = {(double)ar + bg[0] * t, (double)ag + bg[1] * t,
                                 (double)ab + bg[2] * t};
            unsigned char u[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) u[k] = (unsigned char)rint(fmin(fmax(c[k], 0.0), 1.0) * 255.0);
            reinterpret_cast<uchar4 *>(q)[p] = make_uchar4(u[0], u[1], u[2], 255);
        }
        if (final_t) final_t[p] = T;
        if (last_contrib) last_contrib[p] = last;
    }
    if (bt.signal) signal_view_done(bt, fin.view, kSub);
#ifdef G6R_CTA_TRACE
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned k = atomicAdd(&g_cta_trace_n, 1u);
        if (k < (1u << 17)) {
            unsigned smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            g_cta_trace[k][0] = t_start;
            g_cta_trace[k][1] = gtimer();
            g_cta_trace[k][2] = ((unsigned long long)smid << 32) | (unsigned)(fin.view << 16 | (fin.tile * kSub + (fin.band ? 1 : 0)));
            g_cta_trace[k][3] = (unsigned long long)(bt.ws[fin.view].tile_starts[fin.tile + 1] - bt.ws[fin.view].tile_starts[fin.tile]);
        }
    }
#endif
}

// Compositor work order for a batch: every (view, tile) item ranked by its run
// length, longest first (quarter-octave buckets; order inside a bucket is
// arbitrary -- no pixel depends on which CTA composites it or when).  One CTA:
// bucket histogram in shared memory, scan, scatter.  Rank r of the batch lives
// at ws[r / T].sched[r % T]; the compositor's ticket (first view's internal
// slot) is reset here, so the launch needs no cleared workspace.
constexpr int kSchedBuckets = 128;
__device__ __forceinline__ int sched_bucket(int64_t len) {
    if (len <= 0) return kSchedBuckets - 1;   // empty runs last
    const float l2 = __log2f((float)len + 1.0f);
    const int q = (int)(l2 * 4.0f);           // 4 buckets per octave
    return max(0, kSchedBuckets - 2 - q);     // longer -> earlier
}

// With completion signalling (host copies) the order is view by view (longer
// runs first inside a view), so views finish one after another and their
// copies start while later views composite; a run of k times the batch's mean
// length is moved k / 3 - 1 views earlier (at most 8), so a view's long runs
// end about when its short ones do.  (k - 1 views, the earlier rule, prepaid
// so much of the last views' work that they completed in a burst at the end
// of the launch, and their copies trailed it: render_batch on the bench's 20
// views 4.59 -> 4.41 ms; no shift at all measured the same as k / 3.)
constexpr int kViewBuckets = 16;   // one per octave of run length
constexpr int kAllBuckets = kSchedBuckets + kMaxBatch * kViewBuckets;
__device__ __forceinline__ int sched_bucket_prog(int64_t len, int view, int64_t mean, int pnum,
                                                 int pden, int pmax) {
    const int q = len > 0 ? min(kViewBuckets - 1, (int)__log2f((float)len + 1.0f)) : 0;
    const int64_t k = len * pnum / ((mean > 0 ? mean : 1) * pden) - 1;
    const int shift = k < 0 ? 0 : (k > pmax ? pmax : (int)k);
    return kSchedBuckets + max(0, view - shift) * kViewBuckets + (kViewBuckets - 1 - q);
}

__global__ void __launch_bounds__(1024) k_sched_order(const __grid_constant__ Batch bt, int pnum, int pden,
                                                      int pmax) {
    __shared__ unsigned s_cnt[kAllBuckets];
    __shared__ unsigned long long s_sum;
    const int T = bt.vp[0].tiles_x * bt.vp[0].tiles_y;
    const int total = T * bt.nviews;
    const bool prog = bt.signal != 0;
    const int nbk = prog ? kAllBuckets : kSchedBuckets;
    for (int k = threadIdx.x; k < nbk; k += blockDim.x) s_cnt[k] = 0;
    if (threadIdx.x == 0) {
        bt.ws[0].internal[kTicketComposite] = 0;
        s_sum = 0;
    }
    __syncthreads();
    int64_t heavy = 0;
    if (prog) {
        unsigned long long sum = 0;
        for (int i = threadIdx.x; i < total; i += blockDim.x) {
            const int64_t *st = bt.ws[i / T].tile_starts;
            sum += (unsigned long long)(st[i % T + 1] - st[i % T]);
        }
        atomicAdd(&s_sum, sum);
        __syncthreads();
        heavy = (int64_t)(s_sum / (unsigned long long)max(total, 1));   // mean run length
    }
    auto bucket = [&](int i) {
        const int v = i / T, t = i % T;
        const int64_t *st = bt.ws[v].tile_starts;
        const int64_t len = st[t + 1] - st[t];
        return prog ? sched_bucket_prog(len, v, heavy, pnum, pden, pmax) : sched_bucket(len);
    };
    for (int i = threadIdx.x; i < total; i += blockDim.x) atomicAdd(&s_cnt[bucket(i)], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the buckets, one warp
        unsigned carry = 0;
        for (int b0 = 0; b0 < nbk; b0 += 32) {
            const unsigned x = b0 + threadIdx.x < nbk ? s_cnt[b0 + threadIdx.x] : 0u;
            const unsigned inc = warp_inclusive_scan(x);
            if (b0 + threadIdx.x < nbk) s_cnt[b0 + threadIdx.x] = carry + inc - x;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const int v = i / T, t = i % T;
        const unsigned r = atomicAdd(&s_cnt[bucket(i)], 1u);
        bt.ws[r / T].sched[r % T] = ((unsigned)v << 16) | (unsigned)t;
    }
}

// Pack reference-shaped splat arrays (raster.py:405-408) into payloads.
template <typename Real>
__global__ void k_pack_payload(int64_t m, const Real *means2d, const Real *conics, const Real *colors,
                               const Real *alphas, typename Px<Real>::Payload *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    float ex, ey;
    cull_extents((double)conics[3 * i], (double)conics[3 * i + 1], (double)conics[3 * i + 2],
                 sizeof(Real) == 4 ? 0x1p-23 : 0x1p-52, ex, ey, (double)alphas[i]);
    if constexpr (sizeof(Real) == 4) {
        PayloadF32 p;
        p.a = make_float4(means2d[2 * i], means2d[2 * i + 1], conics[3 * i], conics[3 * i + 1]);
        p.b = make_float4(conics[3 * i + 2], alphas[i], colors[3 * i], colors[3 * i + 1]);
        p.c = make_float4(colors[3 * i + 2], ex, ey, power_floor_f32((float)alphas[i]));
        out[i] = p;
    } else {
        PayloadF64 p;
        p.a = make_double2(means2d[2 * i], means2d[2 * i + 1]);
        p.b = make_double2(conics[3 * i], conics[3 * i + 1]);
        p.c = make_double2(conics[3 * i + 2], alphas[i]);
        p.d = make_double2(colors[3 * i], colors[3 * i + 1]);
        p.e = make_double2(colors[3 * i + 2], (double)ex);
        p.f = make_double2((double)ey, power_floor((double)alphas[i]));
        out[i] = p;
    }
}

// Adjoint (f64) of the kernel-module contract (_kernels.pyx:108-187): per-entry
// gradient rows accumulated (+=) into the caller's entry_grads.  One CTA per
// tile, one thread per pixel, row-major (the reference's py-outer, px-inner
// loop).  The CTA walks the tile's entries back to front in lock step; each
// pixel keeps its own reverse sweep (T rebuilt by division, suffix sums) and
// contributes to entry e only while e < its last_contrib.  The contributions
// to one entry are then added in pixel order by 9 reducer threads (one per
// gradient slot), skipping pixels that did not contribute -- the reference's
// summation order, so the rows are deterministic and bit-identical to it (no
// floating-point atomics).
__global__ void __launch_bounds__(1024)
k_composite_backward(ViewParams vp, const double *__restrict__ means2d,
                     const double *__restrict__ conics, const double *__restrict__ colors,
                     const double *__restrict__ alphas, const int32_t *__restrict__ entry_splat,
                     const int64_t *__restrict__ starts, const double *__restrict__ final_t,
                     const int32_t *__restrict__ last_contrib,
                     const double *__restrict__ grad_image, double *entry_grads,
                     const unsigned long long *__restrict__ exp_tab) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int ts = vp.tile_size;
    const int npix = ts * ts;
    double *s_c = reinterpret_cast<double *>(s_raw);                       // [9][npix]
    unsigned char *s_f = reinterpret_cast<unsigned char *>(s_c + 9 * npix);   // [npix]
    __shared__ unsigned long long s_tab[256];
    __shared__ int s_maxlast;
    for (int k = threadIdx.x; k < 256; k += blockDim.x) s_tab[k] = exp_tab[k];
    if (threadIdx.x == 0) s_maxlast = 0;
    const int tile = blockIdx.x;
    const int t = threadIdx.x;
    const int px = (tile % vp.tiles_x) * ts + t % ts;
    const int py = (tile / vp.tiles_x) * ts + t / ts;
    const bool inside = px < vp.iw && py < vp.ih;
    int last = 0;
    double gr = 0.0, gg = 0.0, gb = 0.0, ga = 0.0, T = 1.0;
    if (inside) {
        const int64_t p = (int64_t)py * vp.iw + px;
        last = last_contrib[p];
        gr = grad_image[4 * p];
        gg = grad_image[4 * p + 1];
        gb = grad_image[4 * p + 2];
        ga = grad_image[4 * p + 3];
        T = final_t[p];
        if (gr == 0.0 && gg == 0.0 && gb == 0.0 && ga == 0.0) last = 0;
    }
    __syncthreads();
    if (last > 0) atomicMax(&s_maxlast, last);
    __syncthreads();
    const int64_t lo = starts[tile];
    const double fx = (double)px, fy = (double)py;
    double sr = 0.0, sg = 0.0, sb = 0.0, sa = 0.0;
    for (int64_t e = lo + s_maxlast - 1; e >= lo; --e) {
        double c[9];
        bool contrib = false;
        if (e < lo + last) {
            const int64_t s = entry_splat[e];
            const double dx = fx - means2d[2 * s];
            const double dy = fy - means2d[2 * s + 1];
            const double qa = conics[3 * s], qb = conics[3 * s + 1], qc = conics[3 * s + 2];
            const double pw = -0.5 * (qa * dx * dx + qc * dy * dy) - qb * dx * dy;
            if (!(pw > 0.0 || pw < -4.5)) {
                const double ge = exp_glibc(pw, s_tab);
                const double ai = alphas[s] * ge;
                if (!(ai < 1.0 / 255.0)) {
                    const double om = 1.0 - ai;
                    T = T / om;
                    const double w = ai * T;
                    const double *col = colors + 3 * s;
                    c[5] = w * gr;
                    c[6] = w * gg;
                    c[7] = w * gb;
                    const double dai = T * (col[0] * gr + col[1] * gg + col[2] * gb + ga) -
                                       (sr * gr + sg * gg + sb * gb + sa * ga) / om;
                    c[8] = ge * dai;
                    const double dp = ai * dai;
                    c[0] = dp * (qa * dx + qb * dy);
                    c[1] = dp * (qc * dy + qb * dx);
                    c[2] = dp * (-0.5 * dx * dx);
                    c[3] = dp * (-dx * dy);
                    c[4] = dp * (-0.5 * dy * dy);
                    sr = sr + col[0] * w;
                    sg = sg + col[1] * w;
                    sb = sb + col[2] * w;
                    sa = sa + w;
                    contrib = true;
                }
            }
        }
        s_f[t] = contrib ? 1 : 0;
        if (contrib)
#pragma unroll
            for (int k = 0; k < 9; ++k) s_c[k * npix + t] = c[k];
        __syncthreads();
        if (t < 9) {   // slot t of entry e: the pixels' terms in row-major order
            double acc = entry_grads[9 * e + t];
            for (int q = 0; q < npix; ++q)
                if (s_f[q]) acc = acc + s_c[t * npix + q];
            entry_grads[9 * e + t] = acc;
        }
        __syncthreads();
    }
}

__global__ void k_debug_expf(int64_t n, const float *x, float *y) {
    __shared__ unsigned long long s_tab[32];
    for (int k = threadIdx.x; k < 32; k += blockDim.x) s_tab[k] = c_expf_tab[k];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = expf_glibc(x[i], s_tab);
}

__global__ void k_debug_exp(int64_t n, const double *x, double *y) {
    __shared__ unsigned long long s_tab[256];
    for (int k = threadIdx.x; k < 256; k += blockDim.x) s_tab[k] = c_exp_tab[k];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = exp_glibc(x[i], s_tab);
}

#ifdef G6R_CTA_TRACE
extern "C" int g6r_debug_cta_trace(unsigned long long *host, int max_rows) {
    unsigned n = 0;
    cudaMemcpyFromSymbol(&n, g_cta_trace_n, sizeof n);
    const int rows = (int)std::min<unsigned>(n, (unsigned)max_rows);
    if (rows > 0) cudaMemcpyFromSymbol(host, g_cta_trace, (size_t)rows * 32);
    const unsigned zero = 0;
    cudaMemcpyToSymbol(g_cta_trace_n, &zero, sizeof zero);
    return rows;
}
#endif

int launch_debug_exp(int64_t n, const double *x, double *y, cudaStream_t st) {
    if (n == 0) return G6R_OK;
    k_debug_exp<<<(unsigned)std::min<int64_t>(ceil_div(n, kBlock), 148 * 16), kBlock, 0, st>>>(n, x, y);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_debug_expf(int64_t n, const float *x, float *y, cudaStream_t st) {
    if (n == 0) return G6R_OK;
    k_debug_expf<<<(unsigned)std::min<int64_t>(ceil_div(n, kBlock), 148 * 16), kBlock, 0, st>>>(n, x, y);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_pack_payload(int64_t m, int precision, const void *means2d, const void *conics,
                        const void *colors, const void *alphas, void *payload, cudaStream_t st) {
    if (m == 0) return G6R_OK;
    const unsigned grid = (unsigned)ceil_div(m, kBlock);
    if (precision)
        k_pack_payload<double><<<grid, kBlock, 0, st>>>(
            m, (const double *)means2d, (const double *)conics, (const double *)colors,
            (const double *)alphas, (PayloadF64 *)payload);
    else
        k_pack_payload<float><<<grid, kBlock, 0, st>>>(
            m, (const float *)means2d, (const float *)conics, (const float *)colors,
            (const float *)alphas, (PayloadF32 *)payload);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

constexpr int kCompositeSub = 2;   // CTAs per 16x16 tile

// f32 band compositor (16x16 tiles, two 16x8 band CTAs) with kG lane groups
template <bool kFast, bool kSched>
static void launch_f32_band(int groups, dim3 grid, const Batch &b, int srt, cudaStream_t st) {
    constexpr int nt = 256 / kCompositeSub;
    switch (groups) {
    case 2: k_composite<float, nt, kCompositeSub, kFast, kSched, 2><<<grid, nt, 0, st>>>(b, srt); break;
    case 4: k_composite<float, nt, kCompositeSub, kFast, kSched, 4><<<grid, nt, 0, st>>>(b, srt); break;
    case 8: k_composite<float, nt, kCompositeSub, kFast, kSched, 8><<<grid, nt, 0, st>>>(b, srt); break;
    default: k_composite<float, nt, kCompositeSub, kFast, kSched, 1><<<grid, nt, 0, st>>>(b, srt); break;
    }
}

int launch_composite(const Batch &b, bool sorted, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    const ViewParams &vp = b.vp[0];
    const int threads = vp.tile_size * vp.tile_size;
    const dim3 grid((unsigned)(vp.tiles_x * vp.tiles_y), (unsigned)b.nviews);
    if (grid.x == 0) return G6R_OK;
    const int srt = sorted ? 1 : 0;
    // longest-run-first work order (16x16 tiles: the kSub band kernels)
    static const int sched_env = [] {   // G6R_SCHED=0 keeps launch order (A/B probe)
        const char *e = getenv("G6R_SCHED");
        return e ? atoi(e) : 1;
    }();
    // Batches only: with one view the launch is bound by its heaviest CTA's
    // latency, and longest-first packs the heavy CTAs onto the same SMs (each
    // then shares its SM with other heavy ones) -- measured 0.35 -> 0.47 ms per
    // single-view composite; on batches it saves 7-8 % (tools/probe_composite.py).
    // lane groups per warp hit list (f32 band kernels): 8 groups of 2x2 pixels.
    // cfg3 (tools/probe_bench_views.py, 10-view batches): composite 0.121 ms
    // per view with one list per warp, 0.107 (2 groups), 0.106 (4), 0.103 (8).
    // G6R_GROUPS=1|2|4|8 overrides (A/B probe).
    static const int groups = [] {
        const char *e = getenv("G6R_GROUPS");
        return e ? atoi(e) : 8;
    }();
    bool sched = sched_env && b.nviews > 1 && vp.tile_size == 16 &&
                 grid.x * kCompositeSub <= 65535;
    for (int v = 0; v < b.nviews; ++v) sched = sched && b.ws[v].sched && b.ws[v].internal;
    if (sched) {
        // G6R_PROG="num,den,max" (A/B probe): a run of k x mean moves
        // k * num / den - 1 views earlier, at most max
        static const int3 prog = [] {
            int3 r = make_int3(1, 3, 8);
            if (const char *e = getenv("G6R_PROG")) sscanf(e, "%d,%d,%d", &r.x, &r.y, &r.z);
            return r;
        }();
        k_sched_order<<<1, 1024, 0, st>>>(b, prog.x, prog.y, prog.z);
        trace_mark("sched_order", st);
    }
    // > 48 KB dynamic smem for large f64 tiles; the attribute is per device
    static std::atomic<unsigned long long> attrs_done{0};
    if (const unsigned long long bit = device_bit(); !(attrs_done.load() & bit)) {
        cudaFuncSetAttribute(k_composite<double, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             2 * 1024 * (int)(sizeof(Px<double>::S) + 4));
        cudaFuncSetAttribute(k_composite<float, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             2 * 1024 * (int)(sizeof(Px<float>::S) + 4));
        attrs_done.fetch_or(bit);
    }
    if (vp.precision) {
        // f64 band kernels: grouped hit lists too (G6R_GROUPS64=1: one list per warp)
        static const int groups64 = [] {
            const char *e = getenv("G6R_GROUPS64");
            return e ? atoi(e) : 8;
        }();
        const dim3 g2(grid.x * kCompositeSub, grid.y);
        constexpr int nt = 256 / kCompositeSub;
        if (vp.tile_size == 16 && sched && groups64 == 8)
            k_composite<double, nt, kCompositeSub, false, true, 8><<<g2, nt, 0, st>>>(b, srt);
        else if (vp.tile_size == 16 && groups64 == 8)
            k_composite<double, nt, kCompositeSub, false, false, 8><<<g2, nt, 0, st>>>(b, srt);
        else if (vp.tile_size == 16 && sched)
            k_composite<double, nt, kCompositeSub, false, true><<<g2, nt, 0, st>>>(b, srt);
        else if (vp.tile_size == 16)
            k_composite<double, nt, kCompositeSub><<<g2, nt, 0, st>>>(b, srt);
        else
            k_composite<double, 0><<<grid, threads, 2 * threads * (sizeof(Px<double>::S) + 4), st>>>(b, srt);
    } else {
        bool fast = vp.exp_mode == 1;
        for (int v = 0; v < b.nviews; ++v) fast = fast && !b.out[v].rgba8;   // served bytes stay exact
        const dim3 g2(grid.x * kCompositeSub, grid.y);
        if (vp.tile_size == 16 && fast && sched)
            launch_f32_band<true, true>(groups, g2, b, srt, st);
        else if (vp.tile_size == 16 && fast)
            launch_f32_band<true, false>(groups, g2, b, srt, st);
        else if (vp.tile_size == 16 && sched)
            launch_f32_band<false, true>(groups, g2, b, srt, st);
        else if (vp.tile_size == 16)
            launch_f32_band<false, false>(groups, g2, b, srt, st);
        else
            k_composite<float, 0><<<grid, threads, 2 * threads * (sizeof(Px<float>::S) + 4), st>>>(b, srt);
    }
    trace_mark("composite", st);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_composite_backward(int64_t m, const double *means2d, const double *conics,
                              const double *colors, const double *alphas,
                              const int32_t *entry_splat, const int64_t *tile_starts,
                              const ViewParams &vp, const double *final_t,
                              const int32_t *last_contrib, const double *grad_image,
                              double *entry_grads, cudaStream_t st) {
    (void)m;
    const int threads = vp.tile_size * vp.tile_size;
    const unsigned grid = (unsigned)(vp.tiles_x * vp.tiles_y);
    if (grid == 0) return G6R_OK;
    const size_t smem = (size_t)threads * (9 * sizeof(double) + 1);
    static std::atomic<unsigned long long> attrs_done{0};
    if (const unsigned long long bit = device_bit(); !(attrs_done.load() & bit)) {
        cudaFuncSetAttribute(k_composite_backward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(1024 * (9 * sizeof(double) + 1)));
        attrs_done.fetch_or(bit);
    }
    const unsigned long long *tab = nullptr;
    if (cudaGetSymbolAddress((void **)&tab, c_exp_tab) != cudaSuccess) return G6R_ECUDA;
    k_composite_backward<<<grid, threads, smem, st>>>(vp, means2d, conics, colors, alphas, entry_splat,
                                                      tile_starts, final_t, last_contrib, grad_image,
                                                      entry_grads, tab);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
