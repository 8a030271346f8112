// g6r_project.cu -- per-view slice + EWA projection + cull + compaction +
// tile duplication, fused into one pass over the scene.
//
// Replaces, for one view:
//   raster.py:229-288  _project_rows (stage1 -> opacity modulation -> stage2 ->
//                      fate bincount -> compaction to kept rows, ascending)
//   _kernels.pyx:190-229 project_stage1, :232-363 project_stage2
//   raster.py:340-375  bin_splats up to the key build (rects, counts, offsets,
//                      duplication in splat order, key = tile<<32 | f32 depth)
// One thread per Gaussian reads its 352-byte prepared record as 22 coalesced
// 16-byte column loads, all issued up front.  A launch covers a batch of views
// (grid = views x Gaussian blocks).  The compaction index and the entry offset
// come from one decoupled-lookback scan across CTAs, so the whole stage is a
// single launch with no host round trip.  All
// arithmetic is IEEE double with the reference's association (-fmad=false);
// the only transcendental, exp(-q/2), is CUDA's correctly-rounded-to-1ulp exp.
#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

struct Splat {
    double u, v;            // means2d
    double ca, cb, cc;      // conic (a, b, c)
    double r, g, b;         // clamped SH colour
    double alpha, depth;
    int32_t rx, ry;
};

// project_stage1 for one row (_kernels.pyx:200-229).  prec6 = (00,11,22,01,02,12).
__device__ __forceinline__ int slice_row(const double *mp, const double *md, const double *A,
                                         const double *Q6, double px, double py, double pz,
                                         double *view, double *madj, double &quad) {
    const double ex = mp[0] - px, ey = mp[1] - py, ez = mp[2] - pz;
    const double len = sqrt(ex * ex + ey * ey + ez * ez);
    if (!(len > 1e-12)) return 1;
    const double rl = 1.0 / len;
    view[0] = ex * rl;
    view[1] = ey * rl;
    view[2] = ez * rl;
    const double g0 = view[0] - md[0], g1 = view[1] - md[1], g2 = view[2] - md[2];
    madj[0] = mp[0] + (A[0] * g0 + A[1] * g1 + A[2] * g2);
    madj[1] = mp[1] + (A[3] * g0 + A[4] * g1 + A[5] * g2);
    madj[2] = mp[2] + (A[6] * g0 + A[7] * g1 + A[8] * g2);
    const double diag = Q6[0] * g0 * g0 + Q6[1] * g1 * g1 + Q6[2] * g2 * g2;
    const double off = Q6[3] * g0 * g1 + Q6[4] * g0 * g2 + Q6[5] * g1 * g2;
    quad = diag + 2.0 * off;
    return 0;
}

__device__ __forceinline__ double clamp01(double c) {
    if (c < 0.0) return 0.0;
    if (c > 1.0) return 1.0;
    return c;
}

// project_stage2 for one row (_kernels.pyx:256-363).  Returns the stage code.
__device__ __forceinline__ int project_row(const double *view, const double *madj,
                                           const double *sh, const double *S,
                                           const ViewParams &vp, double sh_c0, double sh_c1,
                                           Splat &o) {
    const double *R = vp.rot;
    const double wx = madj[0] - vp.pos[0], wy = madj[1] - vp.pos[1], wz = madj[2] - vp.pos[2];
    const double tx = R[0] * wx + R[1] * wy + R[2] * wz;
    const double ty = R[3] * wx + R[4] * wy + R[5] * wz;
    const double tz = R[6] * wx + R[7] * wy + R[8] * wz;
    if (!(tz >= vp.znear && tz <= vp.zfar)) return 3;
    o.r = clamp01(sh_c0 * sh[0] - sh_c1 * view[1] * sh[3] + sh_c1 * view[2] * sh[6]
                  - sh_c1 * view[0] * sh[9] + 0.5);
    o.g = clamp01(sh_c0 * sh[1] - sh_c1 * view[1] * sh[4] + sh_c1 * view[2] * sh[7]
                  - sh_c1 * view[0] * sh[10] + 0.5);
    o.b = clamp01(sh_c0 * sh[2] - sh_c1 * view[1] * sh[5] + sh_c1 * view[2] * sh[8]
                  - sh_c1 * view[0] * sh[11] + 0.5);
    const double f = vp.focal;
    const double iz = 1.0 / tz;
    const double u = f * tx * iz + vp.cx;
    const double v = f * ty * iz + vp.cy;
    double xs = tx * iz;
    if (xs < -vp.lim_x) xs = -vp.lim_x;
    else if (xs > vp.lim_x) xs = vp.lim_x;
    xs = xs * tz;
    double ys = ty * iz;
    if (ys < -vp.lim_y) ys = -vp.lim_y;
    else if (ys > vp.lim_y) ys = vp.lim_y;
    ys = ys * tz;
    const double j00 = f * iz;
    const double j02 = -f * xs * iz * iz;
    const double j12 = -f * ys * iz * iz;
    double B[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        B[r][0] = S[3 * r] * R[0] + S[3 * r + 1] * R[1] + S[3 * r + 2] * R[2];
        B[r][1] = S[3 * r] * R[3] + S[3 * r + 1] * R[4] + S[3 * r + 2] * R[5];
        B[r][2] = S[3 * r] * R[6] + S[3 * r + 1] * R[7] + S[3 * r + 2] * R[8];
    }
    const double m00 = R[0] * B[0][0] + R[1] * B[1][0] + R[2] * B[2][0];
    const double m01 = R[0] * B[0][1] + R[1] * B[1][1] + R[2] * B[2][1];
    const double m02 = R[0] * B[0][2] + R[1] * B[1][2] + R[2] * B[2][2];
    const double m11 = R[3] * B[0][1] + R[4] * B[1][1] + R[5] * B[2][1];
    const double m12 = R[3] * B[0][2] + R[4] * B[1][2] + R[5] * B[2][2];
    const double m22 = R[6] * B[0][2] + R[7] * B[1][2] + R[8] * B[2][2];
    const double k00 = j00 * m00 + j02 * m02;
    const double k01 = j00 * m01 + j02 * m12;
    const double k02 = j00 * m02 + j02 * m22;
    const double k11 = j00 * m11 + j12 * m12;
    const double k12 = j00 * m12 + j12 * m22;
    const double ca = k00 * j00 + k02 * j02 + vp.low_pass;
    const double cb = k01 * j00 + k02 * j12;
    const double cc = k11 * j00 + k12 * j12 + vp.low_pass;
    const double det = ca * cc - cb * cb;
    if (!(isfinite(det) && det > 0.0 && isfinite(u) && isfinite(v))) return 4;
    const double idet = 1.0 / det;
    double rx = ceil(3.0 * sqrt(ca));
    if (rx > 1048576.0) rx = 1048576.0;
    double ry = ceil(3.0 * sqrt(cc));
    if (ry > 1048576.0) ry = 1048576.0;
    const int32_t irx = cast_i32_x86(rx), iry = cast_i32_x86(ry);
    if (!(u + (double)irx >= 0.0 && u - (double)irx <= vp.width - 1.0 &&
          v + (double)iry >= 0.0 && v - (double)iry <= vp.height - 1.0))
        return 5;
    o.u = u;
    o.v = v;
    o.ca = cc * idet;
    o.cb = -cb * idet;
    o.cc = ca * idet;
    o.depth = tz;
    o.rx = irx;
    o.ry = iry;
    return 0;
}

// Tile rectangle of a splat (raster.py:359-364), f64 floor then clip.
__device__ __forceinline__ void tile_rect(double u, double v, int32_t rx, int32_t ry,
                                          const ViewParams &vp, int &x0, int &y0, int &wx,
                                          int &hy) {
    const double ts = (double)vp.tile_size;
    long long a, b, c, d;
    if ((vp.tile_size & (vp.tile_size - 1)) == 0) {   // x / 2^k == x * 2^-k exactly
        const double its = 1.0 / ts;
        a = (long long)floor((u - (double)rx) * its);
        b = (long long)floor((u + (double)rx) * its);
        c = (long long)floor((v - (double)ry) * its);
        d = (long long)floor((v + (double)ry) * its);
    } else {
        a = (long long)floor((u - (double)rx) / ts);
        b = (long long)floor((u + (double)rx) / ts);
        c = (long long)floor((v - (double)ry) / ts);
        d = (long long)floor((v + (double)ry) / ts);
    }
    const long long mx = vp.tiles_x - 1, my = vp.tiles_y - 1;
    a = a < 0 ? 0 : (a > mx ? mx : a);
    b = b < 0 ? 0 : (b > mx ? mx : b);
    c = c < 0 ? 0 : (c > my ? my : c);
    d = d < 0 ? 0 : (d > my ? my : d);
    x0 = (int)a;
    y0 = (int)c;
    wx = (int)(b - a + 1);
    hy = (int)(d - c + 1);
}

// Look-back status: one 64-bit word per CTA, [63:62] flag (1 aggregate,
// 2 inclusive prefix), [61:32] splat count, [31:0] entry count (saturating).
// A single volatile 64-bit store publishes flag and both sums together, so no
// memory fence is needed (a __threadfence here is MEMBAR.SC + L1 invalidate).
constexpr unsigned long long kAggFlag = 1ull << 62, kIncFlag = 2ull << 62;
constexpr unsigned long long kECap = 0xffffffffull;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, long long m,
                                                          long long e) {
    const unsigned long long ec = e < (long long)kECap ? (unsigned long long)e : kECap;
    return flag | ((unsigned long long)m << 32) | ec;
}

// Decoupled look-back over CTAs carrying two sums (splats, entries).
// Returns this CTA's exclusive prefix (pm, pe) in shared memory.
__device__ __forceinline__ void lookback2(int64_t tile, long long bm, long long be,
                                          const Workspace &ws, long long *s_pm,
                                          long long *s_pe) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    unsigned long long *status = ws.proj_status;
    if (tile == 0) {
        if (lane == 0) {
            st_volatile_u64(status, pack_status(kIncFlag, bm, be));
            *s_pm = 0;
            *s_pe = 0;
        }
        return;
    }
    if (lane == 0) st_volatile_u64(status + tile, pack_status(kAggFlag, bm, be));
    // Each probe covers 32 x kLB predecessors (lane l owns distances
    // l*kLB+1 .. l*kLB+kLB).  The inclusive-prefix frontier advances by the
    // probe width per L2 round trip, so a narrow probe, not the work, would
    // bound a launch of thousands of short CTAs.
    constexpr int kLB = 8;
    long long pm = 0, pe = 0;
    int64_t j0 = tile - 1;
    while (true) {
        unsigned long long w[kLB];
#pragma unroll
        for (int k = 0; k < kLB; ++k) {
            const int64_t j = j0 - lane * kLB - k;
            w[k] = j >= 0 ? ld_volatile_u64(status + j) : kIncFlag;
        }
        int kfirst = kLB;
#pragma unroll
        for (int k = 0; k < kLB; ++k) {
            const int64_t j = j0 - lane * kLB - k;
            while (!(w[k] >> 62)) w[k] = ld_volatile_u64(status + j);
        }
#pragma unroll
        for (int k = kLB - 1; k >= 0; --k)
            if ((w[k] >> 62) == 2) kfirst = k;
        long long cm = 0, ce = 0;
#pragma unroll
        for (int k = 0; k < kLB; ++k)
            if (k <= kfirst) {
                cm += (long long)((w[k] >> 32) & 0x3fffffffull);
                ce += (long long)(w[k] & kECap);
            }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, kfirst < kLB);
        const int first = inc_mask ? __ffs(inc_mask) - 1 : 32;
        if (lane > first) cm = ce = 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cm += __shfl_xor_sync(0xffffffffu, cm, o);
            ce += __shfl_xor_sync(0xffffffffu, ce, o);
        }
        pm += cm;
        pe += ce;
        if (inc_mask) break;
        j0 -= 32 * kLB;
    }
    if (lane == 0) {
        st_volatile_u64(status + tile, pack_status(kIncFlag, pm + bm, pe + be));
        *s_pm = pm;
        *s_pe = pe;
    }
}

// Block-wide exclusive scan of two ints; returns totals in *tot_a/*tot_b.
__device__ __forceinline__ void block_scan2(int a, int b, int &ea, int &eb, int *s_wa, int *s_wb,
                                            int &tot_a, int &tot_b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ia = warp_inclusive_scan(a);
    const int ib = warp_inclusive_scan(b);
    if (lane == 31) {
        s_wa[warp] = ia;
        s_wb[warp] = ib;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        int va = lane < nw ? s_wa[lane] : 0;
        int vb = lane < nw ? s_wb[lane] : 0;
        const int sa = warp_inclusive_scan(va);
        const int sb = warp_inclusive_scan(vb);
        if (lane < nw) {
            s_wa[lane] = sa - va;
            s_wb[lane] = sb - vb;
        }
        if (lane == nw - 1) {
            s_wa[32] = sa;
            s_wb[32] = sb;
        }
    }
    __syncthreads();
    ea = s_wa[warp] + ia - a;
    eb = s_wb[warp] + ib - b;
    tot_a = s_wa[32];
    tot_b = s_wb[32];
}

// Per-CTA staging of the kept splats' tile rectangles for the duplication.
struct EmitSmem {
    int eoff[kBlock];   // exclusive entry offset inside the CTA
    int x0[kBlock], y0[kBlock], wx[kBlock];
    float rwx[kBlock];  // 1 / wx, for a division-free row/column split
    unsigned db[kBlock];   // f32 depth bits
    unsigned idx[kBlock];  // entry value: compacted splat index or scene row
    int cnt[kBlock];       // entries of the splat (hybrid emission list)
};

__device__ __forceinline__ void stage_rect(EmitSmem &es, int l, int eoff, int x0, int y0, int wx,
                                           unsigned db, unsigned idx) {
    es.eoff[l] = eoff;
    es.x0[l] = x0;
    es.y0[l] = y0;
    es.wx[l] = wx;
    es.rwx[l] = 1.0f / (float)wx;
    es.db[l] = db;
    es.idx[l] = idx;
}

// Cooperative duplication of this CTA's kept splats into (key, value) entries,
// in ascending splat order with tiles row-major inside each rect (the order
// np.repeat produces in raster.py:369-375).  Entry j of the CTA belongs to the
// largest l with eoff[l] <= j (binary search); the row/column split uses a
// float reciprocal corrected to the exact integer quotient.
__device__ __forceinline__ void emit_entries(int nk, int ne, long long e_base, const EmitSmem &es,
                                             int tiles_x, unsigned long long *keys, unsigned *vals) {
    for (int j = threadIdx.x; j < ne; j += blockDim.x) {
        int lo = 0, hi = nk - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (es.eoff[mid] <= j) lo = mid;
            else hi = mid - 1;
        }
        const int loc = j - es.eoff[lo];
        const int w = es.wx[lo];
        int q = (int)((float)loc * es.rwx[lo]);
        if (q * w > loc) --q;
        else if ((q + 1) * w <= loc) ++q;
        const int ty = es.y0[lo] + q;
        const int tx = es.x0[lo] + (loc - q * w);
        const unsigned long long tile = (unsigned long long)ty * (unsigned)tiles_x + (unsigned)tx;
        G6R_CHECK(tile < (unsigned long long)tiles_x * 65536ull);
        keys[e_base + j] = (tile << 32) | es.db[lo];
        vals[e_base + j] = es.idx[lo];
    }
}

constexpr int kDirectEntries = 8;   // splats with at most this many tiles emit their own entries

// Reduce a CTA's drawn-splat depth bits into the view's extrema (for the radix
// key compression in g6r_sort.cu).  Called by every thread.
__device__ __forceinline__ void depth_extrema(bool kept, unsigned db, unsigned *s_dext) {
    const unsigned hi = __reduce_max_sync(0xffffffffu, kept ? db : 0u);
    const unsigned lo_inv = __reduce_max_sync(0xffffffffu, kept ? ~db : 0u);
    if ((threadIdx.x & 31) == 0 && hi) {
        atomicMax(&s_dext[0], lo_inv);
        atomicMax(&s_dext[1], hi);
    }
}

// grid = (views, ceil(n / 256)): CTA (v, *) projects 256 Gaussians for view v.
// The CTAs of the batch's views for one Gaussian block are adjacent in launch
// order, so views 2..K read the block's records from L2.
//
// kOrdered: splats are compacted in scene order (the SplatBatch contract,
// raster.py:157-170) through a decoupled look-back, and entries carry the
// compacted index -- needed when SplatBatch outputs or per-splat rects are
// requested (render_with_state, the backward pass).  Otherwise (the render
// hot path) payloads stay at their scene row, entries carry the row, and a
// CTA reserves its entry block with one atomic: no chain between CTAs.  The
// entry array is then in CTA-completion order, so equal sort keys are put
// back in row order after the sort (k_ranges), which is the reference's tie
// rule (rows ascend with the compacted index).
//
// kSplatKeys (hot path, unordered): no tile entries at all -- every scene row
// writes one depth key (f32 depth bits, all-ones for rows not drawn) and its
// tile rect, for the splat-level sort in g6r_tiles.cu.
#ifndef G6R_PROJ_MINB
#define G6R_PROJ_MINB 4   // CTAs per SM the projection is compiled for (A/B knob)
#endif
template <bool kF64, bool kOrdered, bool kSplatKeys = false>
__global__ void __launch_bounds__(kBlock, G6R_PROJ_MINB)
k_project(g6r_scene scene, uint32_t mask, const __grid_constant__ Batch b, g6r_splat_out so,
          int write_entries, double sh_c0, double sh_c1) {
    __shared__ int s_tile;
    __shared__ int s_wa[33], s_wb[33];
    __shared__ long long s_pm, s_pe;
    __shared__ unsigned s_fate[6];
    __shared__ EmitSmem es;
    __shared__ unsigned s_dext[2];   // block max of ~depth_bits and of depth_bits
    __shared__ int s_nbig;
    __shared__ unsigned s_tot[2];   // splat-keys mode: drawn splats, entries
    const int v = blockIdx.x;
    const ViewParams &vp = b.vp[v];
    const Workspace &ws = b.ws[v];
    int64_t *counters = b.out[v].counters;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd((unsigned long long *)&ws.internal[kTicketProject], 1ull);
    if (threadIdx.x < 6) s_fate[threadIdx.x] = 0;
    if (threadIdx.x < 2) s_dext[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_nbig = 0;
    if (threadIdx.x < 2) s_tot[threadIdx.x] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t n = scene.n;
    const int64_t i = tile * kBlock + threadIdx.x;
    const double2 *rec = reinterpret_cast<const double2 *>(scene.records);

    int st = 255;
    Splat o;
    int x0 = 0, y0 = 0, wx = 0, hy = 0;
    if (i < n) {
        const unsigned fl = scene.flags[i];
        if (((mask >> (fl & 15u)) & 1u) && !(fl & G6R_FLAG_DEGENERATE)) {
            // two phases: the slice columns (mu_p, mu_d, adjust, precision_dd,
            // opacity, w_norm) first, the projection columns (sigma', sh) only for
            // splats that survive the slice -- fewer live registers, more warps
            double r[G6R_REC_DOUBLES];
#pragma unroll
            for (int c = 0; c < 11; ++c) {
                const double2 q = __ldg(&rec[c * n + i]);
                r[2 * c] = q.x;
                r[2 * c + 1] = q.y;
            }
            {
                const double2 q = __ldg(&rec[21 * n + i]);
                r[42] = q.x;
                r[43] = q.y;
            }
            double view[3], madj[3], quad;
            st = slice_row(r + 0, r + 3, r + 6, r + 15, vp.pos[0], vp.pos[1], vp.pos[2], view, madj,
                           quad);
            if (st == 0) {
                const double w = exp(-0.5 * quad) * r[43];   // opacity modulation (raster.py:259-261)
                double alpha = r[42] * w;
                alpha = alpha > vp.alpha_max ? vp.alpha_max : alpha;   // np.minimum (NaN stays)
                o.alpha = alpha;
                if (!(alpha >= kMinAlpha)) st = 2;
            }
            if (st == 0) {
#pragma unroll
                for (int c = 11; c < 21; ++c) {
                    const double2 q = __ldg(&rec[c * n + i]);
                    r[2 * c] = q.x;
                    r[2 * c + 1] = q.y;
                }
                st = project_row(view, madj, r + 30, r + 21, vp, sh_c0, sh_c1, o);
            }
            if (st == 0) tile_rect(o.u, o.v, o.rx, o.ry, vp, x0, y0, wx, hy);
        }
        if (so.stage) so.stage[i] = (uint8_t)st;
    }
    {   // fate histogram: one shared atomic per distinct fate in the warp
        const unsigned peers = __match_any_sync(0xffffffffu, st);
        if (st < 6 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&s_fate[st], (unsigned)__popc(peers));
    }
    const int kept = st == 0;
    const int cnt = kept ? wx * hy : 0;
    const unsigned db = kept ? __float_as_uint((float)o.depth) : 0u;
    depth_extrema(kept, db, s_dext);
    int lm = 0, le = 0, bm = 0, be = 0;
    long long m_base = 0, e_base = 0;
    if (kSplatKeys) {   // only the CTA totals are needed (no entry block)
        const int wm = __reduce_add_sync(0xffffffffu, kept);
        const int we = __reduce_add_sync(0xffffffffu, cnt);
        if ((threadIdx.x & 31) == 0 && wm) {
            atomicAdd(&s_tot[0], (unsigned)wm);
            atomicAdd(&s_tot[1], (unsigned)we);
        }
    } else {
        block_scan2(kept, cnt, lm, le, s_wa, s_wb, bm, be);
        if (kOrdered) {
            lookback2(tile, bm, be, ws, &s_pm, &s_pe);
        } else if (threadIdx.x == 0) {   // reserve this CTA's entry block; count its splats
            s_pm = 0;
            s_pe = (long long)atomicAdd((unsigned long long *)&counters[G6R_CNT_ENTRIES],
                                        (unsigned long long)be);
            if (bm) atomicAdd((unsigned long long *)&counters[G6R_CNT_DRAWN], (unsigned long long)bm);
        }
        __syncthreads();
        m_base = s_pm;
        e_base = s_pe;
    }
    float cex = 0.f, cey = 0.f;   // the payload's cull extents (reused for the culled rect)
    if (kept) {
        const long long m = kOrdered ? m_base + lm : i;
        if (kF64) {
            float &ex = cex, &ey = cey;
            cull_extents(o.ca, o.cb, o.cc, 0x1p-52, ex, ey, o.alpha);
            PayloadF64 p;
            p.a = make_double2(o.u, o.v);
            p.b = make_double2(o.ca, o.cb);
            p.c = make_double2(o.cc, o.alpha);
            p.d = make_double2(o.r, o.g);
            p.e = make_double2(o.b, (double)ex);
            p.f = make_double2((double)ey, power_floor(o.alpha));
            reinterpret_cast<PayloadF64 *>(ws.payload)[m] = p;
        } else {
            const float fa = (float)o.ca, fb = (float)o.cb, fc = (float)o.cc;
            float &ex = cex, &ey = cey;
            const float fal = (float)o.alpha;
            cull_extents_f32(fa, fb, fc, ex, ey, fal);
            PayloadF32 p;
            p.a = make_float4((float)o.u, (float)o.v, fa, fb);
            p.b = make_float4(fc, fal, (float)o.r, (float)o.g);
            p.c = make_float4((float)o.b, ex, ey, power_floor_f32(fal));
            reinterpret_cast<PayloadF32 *>(ws.payload)[m] = p;
        }
        if (kOrdered) {
        if (so.gids) so.gids[m] = i;
        if (so.means2d) {
            so.means2d[2 * m] = o.u;
            so.means2d[2 * m + 1] = o.v;
        }
        if (so.conics) {
            so.conics[3 * m] = o.ca;
            so.conics[3 * m + 1] = o.cb;
            so.conics[3 * m + 2] = o.cc;
        }
        if (so.colors) {
            so.colors[3 * m] = o.r;
            so.colors[3 * m + 1] = o.g;
            so.colors[3 * m + 2] = o.b;
        }
        if (so.alphas) so.alphas[m] = o.alpha;
        if (so.depths) so.depths[m] = o.depth;
        if (so.radii) {
            so.radii[2 * m] = o.rx;
            so.radii[2 * m + 1] = o.ry;
        }
        }
        if (kOrdered && ws.splat_rect) ws.splat_rect[m] = make_int4((int)(e_base + le), x0, y0, wx);
    }
    if (kSplatKeys) {
        if (i < n) {
            ws.keys[0][i] = kept ? (unsigned long long)db : 0xffffffffull;
            ws.rect[i] = kept ? make_uint2((unsigned)x0 | ((unsigned)y0 << 16),
                                           (unsigned)wx | ((unsigned)hy << 16))
                              : make_uint2(0u, 0u);
            // The tiles of the rect that the compositor's cull box touches:
            // pixel columns [ceil(fl(mx - ex)), floor(fl(mx + ex))] -- the same
            // float tests as the compositor's (g6r_composite.cu stage) --
            // clipped to the image.  Entries outside it are never visited by
            // any pixel, so runs without exported indices skip them.
            uint2 cr = make_uint2(0u, 0u);
            if (kept) {
                const float ex = cex, ey = cey;
                const float mxf = (float)o.u, myf = (float)o.v;
                const int ts = vp.tile_size;
                const int xl = max(__float2int_ru(mxf - ex), 0), xh = min(__float2int_rd(mxf + ex), vp.iw - 1);
                const int yl = max(__float2int_ru(myf - ey), 0), yh = min(__float2int_rd(myf + ey), vp.ih - 1);
                if (xl <= xh && yl <= yh) {
                    // pixel -> tile (non-negative): a shift for power-of-two tiles
                    const bool pow2 = (ts & (ts - 1)) == 0;
                    const int sh = __ffs(ts) - 1;
                    auto tdiv = [&](int p) { return pow2 ? p >> sh : p / ts; };
                    const int cx0 = max(tdiv(xl), x0), cx1 = min(tdiv(xh), x0 + wx - 1);
                    const int cy0 = max(tdiv(yl), y0), cy1 = min(tdiv(yh), y0 + hy - 1);
                    if (cx0 <= cx1 && cy0 <= cy1)
                        cr = make_uint2((unsigned)cx0 | ((unsigned)cy0 << 16),
                                        (unsigned)(cx1 - cx0 + 1) | ((unsigned)(cy1 - cy0 + 1) << 16));
                }
            }
            ws.crect[i] = cr;
        }
        __syncthreads();
        // this block's drawn count, for the optional export of the runs as
        // compacted splat indices (k_rank_scan / k_rank_fill, g6r_tiles.cu)
        if (threadIdx.x == 0 && s_tot[0]) ws.proj_status[tile] = s_tot[0];
        if (threadIdx.x == 0 && s_tot[0]) {
            atomicAdd((unsigned long long *)&counters[G6R_CNT_DRAWN], (unsigned long long)s_tot[0]);
            atomicAdd((unsigned long long *)&counters[G6R_CNT_ENTRIES], (unsigned long long)s_tot[1]);
        }
        if (threadIdx.x < 6 && s_fate[threadIdx.x])
            atomicAdd((unsigned long long *)&counters[G6R_CNT_FATE + threadIdx.x],
                      (unsigned long long)s_fate[threadIdx.x]);
        if (threadIdx.x == 0 && s_dext[1]) note_depth_extrema(ws.internal, s_dext[0], s_dext[1]);
        return;
    }
    // Duplication, hybrid: a splat with few tiles writes its own entries (row-
    // major over its rect); larger ones are queued and emitted by the whole CTA.
    const bool emit_ok = write_entries && e_base + be <= ws.entry_capacity;
    if (kept && emit_ok) {
        const long long m = kOrdered ? m_base + lm : i;
        if (cnt <= kDirectEntries) {
            G6R_CHECK(e_base + le + cnt <= ws.entry_capacity);
            unsigned long long *keys = ws.keys[0] + e_base + le;
            unsigned *vals = ws.vals[0] + e_base + le;
            int k = 0;
            for (int yy = 0; yy < hy; ++yy)
                for (int xx = 0; xx < wx; ++xx, ++k) {
                    const unsigned long long t =
                        (unsigned long long)(y0 + yy) * (unsigned)vp.tiles_x + (unsigned)(x0 + xx);
                    keys[k] = (t << 32) | db;
                    vals[k] = (unsigned)m;
                }
        } else {
            const int q = atomicAdd(&s_nbig, 1);
            stage_rect(es, q, le, x0, y0, wx, db, (unsigned)m);
            es.cnt[q] = cnt;
        }
    }
    __syncthreads();
    if (threadIdx.x < 6 && s_fate[threadIdx.x])
        atomicAdd((unsigned long long *)&counters[G6R_CNT_FATE + threadIdx.x],
                  (unsigned long long)s_fate[threadIdx.x]);
    if (threadIdx.x == 0 && s_dext[1]) note_depth_extrema(ws.internal, s_dext[0], s_dext[1]);
    if (emit_ok) {
        const int nbig = s_nbig;
        for (int q = 0; q < nbig; ++q) {   // queued large rects, all threads per rect
            const int n_e = es.cnt[q], w = es.wx[q], base = es.eoff[q];
            const float rw = es.rwx[q];
            for (int k = threadIdx.x; k < n_e; k += blockDim.x) {
                int r = (int)((float)k * rw);
                if (r * w > k) --r;
                else if ((r + 1) * w <= k) ++r;
                const unsigned long long t = (unsigned long long)(es.y0[q] + r) * (unsigned)vp.tiles_x +
                                             (unsigned)(es.x0[q] + (k - r * w));
                G6R_CHECK(e_base + base + k < ws.entry_capacity);
                ws.keys[0][e_base + base + k] = (t << 32) | es.db[q];
                ws.vals[0][e_base + base + k] = es.idx[q];
            }
        }
    } else if (write_entries && threadIdx.x == 0) {
        counters[G6R_CNT_OVERFLOW] = 1;
    }
    if (kOrdered && tile == gridDim.y - 1 && threadIdx.x == 0) {
        counters[G6R_CNT_DRAWN] = m_base + bm;
        counters[G6R_CNT_ENTRIES] = e_base + be;
    }
}

// Binning of externally supplied splats (raster.py:340-375 on a given
// SplatBatch), one view.
__global__ void __launch_bounds__(kBlock)
k_duplicate(int64_t m, const double *__restrict__ means2d, const int32_t *__restrict__ radii,
            const double *__restrict__ depths, const __grid_constant__ Batch b) {
    __shared__ int s_tile;
    __shared__ int s_wa[33], s_wb[33];
    __shared__ long long s_pm, s_pe;
    __shared__ EmitSmem es;
    __shared__ unsigned s_dext[2];
    const ViewParams &vp = b.vp[0];
    const Workspace &ws = b.ws[0];
    int64_t *counters = b.out[0].counters;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd((unsigned long long *)&ws.internal[kTicketProject], 1ull);
    if (threadIdx.x < 2) s_dext[threadIdx.x] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t i = tile * kBlock + threadIdx.x;
    int x0 = 0, y0 = 0, wx = 0, hy = 0;
    const int kept = i < m;
    if (kept) tile_rect(means2d[2 * i], means2d[2 * i + 1], radii[2 * i], radii[2 * i + 1], vp, x0, y0, wx, hy);
    const int cnt = kept ? wx * hy : 0;
    const unsigned db = kept ? __float_as_uint((float)depths[i]) : 0u;
    depth_extrema(kept, db, s_dext);
    int lm, le, bm, be;
    block_scan2(kept, cnt, lm, le, s_wa, s_wb, bm, be);
    lookback2(tile, bm, be, ws, &s_pm, &s_pe);
    __syncthreads();
    const long long m_base = s_pm, e_base = s_pe;
    if (kept) stage_rect(es, lm, le, x0, y0, wx, db, (unsigned)(m_base + lm));
    __syncthreads();
    if (threadIdx.x == 0 && s_dext[1]) note_depth_extrema(ws.internal, s_dext[0], s_dext[1]);
    if (e_base + be <= ws.entry_capacity) {
        emit_entries(bm, be, e_base, es, vp.tiles_x, ws.keys[0], ws.vals[0]);
    } else if (threadIdx.x == 0) {
        counters[G6R_CNT_OVERFLOW] = 1;
    }
    if (tile == gridDim.x - 1 && threadIdx.x == 0) {
        counters[G6R_CNT_DRAWN] = m;
        counters[G6R_CNT_ENTRIES] = e_base + be;
    }
}

// --- kernel-module contract mirrors (uncompacted, per row) ----------------------
__global__ void k_stage1(int64_t n, const double *mu_p, const double *mu_d, const double *adjust,
                         const double *prec, double px, double py, double pz, double *view,
                         double *mean_adj, double *quad, uint8_t *stage) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *Q = prec + 9 * i;
    const double q6[6] = {Q[0], Q[4], Q[8], Q[1], Q[2], Q[5]};
    double v[3], ma[3], q;
    if (slice_row(mu_p + 3 * i, mu_d + 3 * i, adjust + 9 * i, q6, px, py, pz, v, ma, q)) {
        stage[i] = 1;
        return;
    }
    for (int k = 0; k < 3; ++k) {
        view[3 * i + k] = v[k];
        mean_adj[3 * i + k] = ma[k];
    }
    quad[i] = q;
}

__global__ void k_stage2(int64_t n, const double *view, const double *mean_adj, const double *sh,
                         const double *sigma_prime, ViewParams vp, double sh_c0, double sh_c1,
                         double *means2d, double *conics, double *colors, double *depths,
                         int32_t *radii, uint8_t *stage) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || stage[i] != 0) return;
    Splat o;
    const int st = project_row(view + 3 * i, mean_adj + 3 * i, sh + 12 * i, sigma_prime + 9 * i,
                               vp, sh_c0, sh_c1, o);
    if (st) {
        stage[i] = (uint8_t)st;
        return;
    }
    means2d[2 * i] = o.u;
    means2d[2 * i + 1] = o.v;
    conics[3 * i] = o.ca;
    conics[3 * i + 1] = o.cb;
    conics[3 * i + 2] = o.cc;
    colors[3 * i] = o.r;
    colors[3 * i + 1] = o.g;
    colors[3 * i + 2] = o.b;
    depths[i] = o.depth;
    radii[2 * i] = o.rx;
    radii[2 * i + 1] = o.ry;
}

static const double kShC0 = 0.28209479177387814;   // core.py:25
static const double kShC1 = 0.4886025119029199;    // core.py:26

bool projection_ordered(const Batch &b, const g6r_splat_out *splats, bool write_entries) {
    if (!write_entries || b.ws[0].splat_rect) return true;
    return splats && (splats->gids || splats->means2d || splats->conics || splats->colors ||
                      splats->alphas || splats->depths || splats->radii || splats->stage);
}

bool splat_sort_applies(const Batch &b) {
    return (int64_t)b.vp[0].tiles_x * b.vp[0].tiles_y <= kMaxSplatSortTiles;
}

int launch_project(const g6r_scene &scene, uint32_t mask, const Batch &b,
                   const g6r_splat_out *splats, bool write_entries, cudaStream_t st) {
    g6r_splat_out so{};
    if (splats) so = *splats;
    if (scene.n == 0 || b.nviews == 0) return G6R_OK;
    const dim3 grid((unsigned)b.nviews, (unsigned)ceil_div(scene.n, kBlock));
    // compacted (ordered) only when SplatBatch-shaped outputs or rects are wanted
    const bool ordered = projection_ordered(b, splats, write_entries);
    const bool keys = !ordered && splat_sort_applies(b);
    const bool f64 = b.vp[0].precision != 0;
    if (f64 && ordered)
        k_project<true, true><<<grid, kBlock, 0, st>>>(scene, mask, b, so, write_entries, kShC0, kShC1);
    else if (f64 && keys)
        k_project<true, false, true><<<grid, kBlock, 0, st>>>(scene, mask, b, so, write_entries, kShC0, kShC1);
    else if (f64)
        k_project<true, false><<<grid, kBlock, 0, st>>>(scene, mask, b, so, write_entries, kShC0, kShC1);
    else if (ordered)
        k_project<false, true><<<grid, kBlock, 0, st>>>(scene, mask, b, so, write_entries, kShC0, kShC1);
    else if (keys)
        k_project<false, false, true><<<grid, kBlock, 0, st>>>(scene, mask, b, so, write_entries, kShC0, kShC1);
    else
        k_project<false, false><<<grid, kBlock, 0, st>>>(scene, mask, b, so, write_entries, kShC0, kShC1);
    trace_mark("project", st);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_duplicate(int64_t m, const double *means2d, const int32_t *radii, const double *depths,
                     const Batch &b, cudaStream_t st) {
    if (m == 0) return G6R_OK;
    k_duplicate<<<(unsigned)ceil_div(m, kBlock), kBlock, 0, st>>>(m, means2d, radii, depths, b);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_stage1(int64_t n, const double *mu_p, const double *mu_d, const double *adjust,
                  const double *prec, double px, double py, double pz, double *view,
                  double *mean_adj, double *quad, uint8_t *stage, cudaStream_t st) {
    if (n == 0) return G6R_OK;
    k_stage1<<<(unsigned)ceil_div(n, kBlock), kBlock, 0, st>>>(n, mu_p, mu_d, adjust, prec, px, py,
                                                                pz, view, mean_adj, quad, stage);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_stage2(int64_t n, const double *view, const double *mean_adj, const double *sh,
                  const double *sigma_prime, const double *rot, double px, double py, double pz,
                  double znear, double zfar, double f, double ox, double oy, double lim_x,
                  double lim_y, double width, double height, double low_pass, double sh_c0,
                  double sh_c1, double *means2d, double *conics, double *colors, double *depths,
                  int32_t *radii, uint8_t *stage, cudaStream_t st) {
    if (n == 0) return G6R_OK;
    ViewParams vp{};
    vp.pos[0] = px;
    vp.pos[1] = py;
    vp.pos[2] = pz;
    for (int k = 0; k < 9; ++k) vp.rot[k] = rot[k];
    vp.focal = f;
    vp.cx = ox;
    vp.cy = oy;
    vp.znear = znear;
    vp.zfar = zfar;
    vp.lim_x = lim_x;
    vp.lim_y = lim_y;
    vp.width = width;
    vp.height = height;
    vp.low_pass = low_pass;
    k_stage2<<<(unsigned)ceil_div(n, kBlock), kBlock, 0, st>>>(n, view, mean_adj, sh, sigma_prime,
                                                                vp, sh_c0, sh_c1, means2d, conics,
                                                                colors, depths, radii, stage);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
