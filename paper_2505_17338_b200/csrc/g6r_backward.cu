// g6r_backward.cu -- analytic gradients of the render path (f64), on device.
//
// Replaces diffrender.py:401-439 render_backward:
//   composite_backward (_kernels.pyx:108-187)  -> k_composite_bwd
//   np.add.at(g_splat, entry_splat, entry_grads) (diffrender.py:436-437)
//                                              -> k_splat_grad_sum
//   _backward_rows (diffrender.py:183-398)     -> k_backward_rows
// Deterministic by construction (no floating-point atomics): every entry's
// gradient row is reduced over the tile's pixels in a fixed order (a transposed
// sum through shared memory inside a warp, warps in index order) and written once, to the entry's
// pre-sort slot; a splat's rows are then summed sequentially in ascending tile
// order -- the order np.add.at visits them in the reference.  Results match
// the reference to rounding (different association of the pixel sums), not
// bit for bit.
#include <algorithm>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

#ifndef G6R_BWD_BATCH
#define G6R_BWD_BATCH 64
#endif
// G6R_BWD_RCP: T / om and the suffix term / om share one reciprocal of om
// (a few ulp from the reference's two divisions, well inside the backward's
// rtol 1e-7; fine-tune 3.55 -> 3.45 ms/iter).  0 restores the two divisions.
#ifndef G6R_BWD_RCP
#define G6R_BWD_RCP 1
#endif
constexpr int kBwdBatch = G6R_BWD_BATCH;   // entries staged per backward batch
constexpr int kBwdWords = kBwdBatch / 32;     // hit-mask words per warp and batch
static_assert(kBwdBatch % 32 == 0 && kBwdBatch <= 128, "batch: whole warps, one entry per thread");

struct BwdSplat {
    double mx, my, ca, cb, cc, alpha, r, g, b;
};

// Two CTAs per tile, one per 16x8 band (8x4 warp blocks, as the forward), one
// thread per pixel; each band sweeps the run back to front from its own largest
// last_contrib and writes its own row per entry (egrad + band * cap * 9).
// Each warp walks only the batch entries whose footprint meets its 8x4 block
// (a ballot of the staged masks, set bits in ascending order: the entry order
// of the sweep), and records which of them it gave a nonzero row.
__constant__ unsigned long long c_bwd_exp_tab[256] = G6R_EXP_TABLE;

__global__ void __launch_bounds__(128)
k_composite_bwd(ViewParams vp, const PayloadF64 *__restrict__ payload,
                const unsigned *vals0, const unsigned *vals1, const long long *internal,
                const int64_t *__restrict__ starts, const double *__restrict__ final_t,
                const int32_t *__restrict__ last_contrib, const double *__restrict__ grad_image,
                const int4 *__restrict__ rect, double *__restrict__ egrad_all, int64_t cap) {
    __shared__ BwdSplat s_sp[kBwdBatch];
    __shared__ int s_orig[2][kBwdBatch];   // by batch parity: staged while the previous is written
    __shared__ unsigned s_mask[kBwdBatch];
    __shared__ double s_part[4][kBwdBatch][9];
    __shared__ double s_red[4][9][33];   // per-warp transpose of the 9 partials
    __shared__ unsigned s_rowm[4][kBwdWords];   // per warp: entries with a nonzero row
    __shared__ float4 s_wbox[4];
    __shared__ int s_maxlast;
    __shared__ unsigned long long s_etab[256];   // glibc exp table (g6r_common.cuh)
    for (int k = threadIdx.x; k < 256; k += blockDim.x) s_etab[k] = c_bwd_exp_tab[k];
    const int ts = 16;
    const int tile = blockIdx.x >> 1, band = (int)(blockIdx.x & 1) * 8;
    double *__restrict__ egrad = egrad_all + (int64_t)(blockIdx.x & 1) * cap * 9;
    const int tx = tile % vp.tiles_x, ty = tile / vp.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * ts + (warp & 1) * 8 + (lane & 7);
    const int py = ty * ts + band + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = px < vp.iw && py < vp.ih;
    if (threadIdx.x < 4) {
        const int w = threadIdx.x;
        const int x0 = tx * ts + (w & 1) * 8, y0 = ty * ts + band + (w >> 1) * 4;
        const int x1 = min(x0 + 7, vp.iw - 1), y1 = min(y0 + 3, vp.ih - 1);
        s_wbox[w] = (x0 <= x1 && y0 <= y1) ? make_float4((float)x0, (float)x1, (float)y0, (float)y1)
                                           : make_float4(1e30f, -1e30f, 1e30f, -1e30f);
    }
    if (threadIdx.x == 0) s_maxlast = 0;
    const unsigned *vals = (internal && sorted_buffer(internal)) ? vals1 : vals0;
    const int64_t lo = starts[tile], hi = starts[tile + 1];
    int last = 0;
    double T = 1.0, gr = 0.0, gg = 0.0, gb = 0.0, ga = 0.0;
    bool active = false;
    if (inside) {
        const int64_t p = (int64_t)py * vp.iw + px;
        last = last_contrib[p];
        gr = grad_image[4 * p];
        gg = grad_image[4 * p + 1];
        gb = grad_image[4 * p + 2];
        ga = grad_image[4 * p + 3];
        T = final_t[p];
        active = last > 0 && !(gr == 0.0 && gg == 0.0 && gb == 0.0 && ga == 0.0);
    }
    __syncthreads();
    if (active) atomicMax(&s_maxlast, last);
    __syncthreads();
    const int64_t top = lo + s_maxlast;
    const double fx = (double)px, fy = (double)py;
    double sr = 0.0, sg = 0.0, sb = 0.0, sa = 0.0;
    // Stage the batch ending at b (entries b-1 down to b-cnt): splat rows, the
    // entries' egrad slots, per-warp footprint masks.  `m` is this thread's
    // entry's splat row, loaded one batch ahead (its latency hides behind the
    // previous batch's sweep).
    auto batch_len = [&](int64_t b) { return (int)(b - lo < kBwdBatch ? b - lo : kBwdBatch); };
    auto fetch_row = [&](int64_t b) {
        return (b > lo && threadIdx.x < batch_len(b)) ? vals[b - 1 - threadIdx.x] : 0u;
    };
    auto stage = [&](int64_t b, int buf, unsigned m) {
        if (b <= lo || threadIdx.x >= batch_len(b)) return;
        const int j = threadIdx.x;
        const PayloadF64 pl = payload[m];
        s_sp[j] = BwdSplat{pl.a.x, pl.a.y, pl.b.x, pl.b.y, pl.c.x, pl.c.y, pl.d.x, pl.d.y, pl.e.x};
        const int4 rc = rect[m];
        s_orig[buf][j] = rc.x + (ty - rc.z) * rc.w + (tx - rc.y);
        const float ex = (float)pl.e.y, ey = (float)pl.f.x;
        const float mx = (float)pl.a.x, my = (float)pl.a.y;
        unsigned mk = 0;
        for (int w = 0; w < 4; ++w) {
            const float4 bx = s_wbox[w];
            if (mx + ex >= bx.x && mx - ex <= bx.y && my + ey >= bx.z && my - ey <= bx.w) mk |= 1u << w;
        }
        s_mask[j] = mk;
    };
    stage(top, 0, fetch_row(top));
    unsigned m_next = fetch_row(top - kBwdBatch);
    __syncthreads();
    int buf = 0;
    for (int64_t b1 = top; b1 > lo; b1 -= kBwdBatch, buf ^= 1) {
        const int cnt = batch_len(b1);
        unsigned hitw[kBwdWords], rowm[kBwdWords];
#pragma unroll
        for (int q = 0; q < kBwdWords; ++q) {
            const int j = q * 32 + lane;
            hitw[q] = __ballot_sync(0xffffffffu, j < cnt && ((s_mask[j] >> warp) & 1u));
            rowm[q] = 0u;
        }
#pragma unroll
        for (int q = 0; q < kBwdWords; ++q) while (hitw[q]) {   // warp-uniform: the entries some pixel of this warp may reach
            const int j = q * 32 + __ffs(hitw[q]) - 1;
            hitw[q] &= hitw[q] - 1u;
            const int64_t e = b1 - 1 - j;
            double c[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) c[k] = 0.0;
            bool contrib = false;
            if (active && e < lo + last) {
                const BwdSplat s = s_sp[j];
                const double dx = fx - s.mx, dy = fy - s.my;
                const double pw = -0.5 * (s.ca * dx * dx + s.cc * dy * dy) - s.cb * dx * dy;
                if (!(pw > 0.0 || pw < -4.5)) {
                    const double ge = exp_glibc(pw, s_etab);   // libm exp (_kernels.pyx:172)
                    const double ai = s.alpha * ge;
                    if (!(ai < 1.0 / 255.0)) {
                        const double om = 1.0 - ai;
#if G6R_BWD_RCP
                        const double rom = 1.0 / om;   // one division for T and the suffix term
                        T = T * rom;
#else
                        T = T / om;
#endif
                        const double w = ai * T;
                        c[5] = w * gr;
                        c[6] = w * gg;
                        c[7] = w * gb;
#if G6R_BWD_RCP
                        const double dai = T * (s.r * gr + s.g * gg + s.b * gb + ga) -
                                           (sr * gr + sg * gg + sb * gb + sa * ga) * rom;
#else
                        const double dai = T * (s.r * gr + s.g * gg + s.b * gb + ga) -
                                           (sr * gr + sg * gg + sb * gb + sa * ga) / om;
#endif
                        c[8] = ge * dai;
                        const double dp = ai * dai;
                        c[0] = dp * (s.ca * dx + s.cb * dy);
                        c[1] = dp * (s.cc * dy + s.cb * dx);
                        c[2] = dp * (-0.5 * dx * dx);
                        c[3] = dp * (-dx * dy);
                        c[4] = dp * (-0.5 * dy * dy);
                        sr = sr + s.r * w;
                        sg = sg + s.g * w;
                        sb = sb + s.b * w;
                        sa = sa + w;
                        contrib = true;
                    }
                }
            }
            if (!__any_sync(0xffffffffu, contrib)) continue;   // an exact zero row: no reduction
            rowm[q] |= 1u << (j & 31);
            // transpose through shared memory: lane 3k+p sums 11 (p < 2) or 10
            // lanes' values of component k in lane order, then p = 0 adds the
            // other two parts -- a fixed order (deterministic), ~40 issue slots
            // instead of 9 xor-shuffle trees of f64 (~135)
            double *red = &s_red[warp][0][0];
#pragma unroll
            for (int k = 0; k < 9; ++k) red[k * 33 + lane] = c[k];
            __syncwarp();
            double part = 0.0;
            const int rk = lane / 3, rp = lane - 3 * (lane / 3);
            if (lane < 27) {
                const double *row = red + rk * 33 + rp * 11;
                const int len = rp < 2 ? 11 : 10;
                part = row[0];
                for (int q = 1; q < len; ++q) part += row[q];
            }
            const double p1 = __shfl_down_sync(0xffffffffu, part, 1);
            const double p2 = __shfl_down_sync(0xffffffffu, part, 2);
            if (lane < 27 && rp == 0) s_part[warp][j][rk] = (part + p1) + p2;
            __syncwarp();
        }
        if (lane < kBwdWords) {
            unsigned v = rowm[0];
#pragma unroll
            for (int q = 1; q < kBwdWords; ++q)
                if (lane == q) v = rowm[q];
            s_rowm[warp][lane] = v;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < cnt * 9; q += blockDim.x) {   // warps in index order
            const int j = q / 9, k = q % 9;
            double v = 0.0;
            for (int w = 0; w < 4; ++w)
                if ((s_rowm[w][j >> 5] >> (j & 31)) & 1u) v += s_part[w][j][k];
            G6R_CHECK(s_orig[buf][j] >= 0 && s_orig[buf][j] < cap);
            egrad[(int64_t)s_orig[buf][j] * 9 + k] = v;
        }
        // the next batch is staged in the same phase (its buffers are not read here)
        stage(b1 - kBwdBatch, buf ^ 1, m_next);
        m_next = fetch_row(b1 - 2 * kBwdBatch);
        __syncthreads();
    }
}

// Zero both bands' rows of the view's entries (slots [0, entries)): rows the
// sweep never reaches stay zero; the rest are overwritten.  Also clears the
// per-row drawn marks (k_splat_grad_sum sets the view's drawn rows).
__global__ void k_zero_rows(const int64_t *counters, int64_t cap, double *__restrict__ egrad,
                            int64_t scene_rows, uint8_t *__restrict__ drawn) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < scene_rows;
         i += (int64_t)gridDim.x * blockDim.x)
        drawn[i] = 0;
    const int64_t e = counters[G6R_CNT_ENTRIES];
    const int64_t n = (e < cap ? e : cap) * 9;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        egrad[i] = 0.0;
        egrad[cap * 9 + i] = 0.0;
    }
}

// g_splat of drawn splat m = sum of its entries' rows, ascending tile order
// (np.add.at order), stored at its scene row gids[m], which is marked drawn.
__global__ void k_splat_grad_sum(int64_t m_total, const int4 *__restrict__ rect,
                                 const int64_t *counters, const double *__restrict__ egrad,
                                 int64_t cap, const int64_t *__restrict__ gids,
                                 double *__restrict__ gsplat, uint8_t *__restrict__ drawn) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t mm = counters[G6R_CNT_DRAWN];
    // an overflowed forward (entries beyond the capacity, empty runs) has no
    // entry rows: every splat stays undrawn, so every gradient row is zero
    if (counters[G6R_CNT_OVERFLOW] || m >= mm || m >= m_total) return;
    const int64_t a = rect[m].x;
    const int64_t b = m + 1 < mm ? (int64_t)rect[m + 1].x : counters[G6R_CNT_ENTRIES];
    double acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.0;
    for (int64_t i = a; i < b; ++i)   // entry row = upper band + lower band
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += egrad[i * 9 + k] + egrad[(cap + i) * 9 + k];
    const int64_t row = gids[m];
    G6R_CHECK(row >= 0 && row < m_total && a <= b && b <= cap);
#pragma unroll
    for (int k = 0; k < 9; ++k) gsplat[row * 9 + k] = acc[k];
    drawn[row] = 1;
}

struct BwdScene {
    const double *mu_p, *mu_d, *cov_raw, *sh;
    double ss[3], ds;
    int w_mode;
};

struct BwdOut {
    double *g_mu_p, *g_mu_d, *g_cov_raw, *g_sh, *g_opacity_raw;
};

#ifndef G6R_ROWS_MINB
#define G6R_ROWS_MINB 3
#endif
// Chain one drawn splat's 9 screen-space gradients gs to its 40 raw
// parameters (diffrender.py:183-398, same intermediate names): go = g_mu_p (3),
// g_mu_d (3), g_cov_raw (21, from the row's raw cov parameters `raw`), g_sh
// (12), g_opacity_raw (1).
constexpr int kGradOut = 40;
__device__ __forceinline__ void chain_row(const ViewParams &vp, const BwdScene &sc,
                                          const double2 *__restrict__ rec, int64_t n, int64_t i,
                                          const double *raw, const double *gs, double sh_c0,
                                          double sh_c1, double *go) {
    double r[G6R_REC_DOUBLES];
#pragma unroll
    for (int c = 0; c < G6R_REC_COLUMNS; ++c) {
        const double2 q = rec[c * n + i];
        r[2 * c] = q.x;
        r[2 * c + 1] = q.y;
    }
    const double *adj = r + 6;   // 3x3 row-major
    const double Q[3][3] = {{r[15], r[18], r[19]}, {r[18], r[16], r[20]}, {r[19], r[20], r[17]}};
    const double *sp = r + 21;   // sigma' 3x3 row-major
    const double *shc = r + 30;
    const double opacity = r[42], w_norm = r[43];
    const double *R = vp.rot;
    const double f = vp.focal;
    const double *mp = sc.mu_p + 3 * i, *md = sc.mu_d + 3 * i;

    // --- forward replay -----------------------------------------------------
    const double dxw = mp[0] - vp.pos[0], dyw = mp[1] - vp.pos[1], dzw = mp[2] - vp.pos[2];
    const double dist = sqrt(dxw * dxw + dyw * dyw + dzw * dzw);
    const double inv_dist = 1.0 / dist;
    const double v[3] = {dxw * inv_dist, dyw * inv_dist, dzw * inv_dist};
    const double d[3] = {v[0] - md[0], v[1] - md[1], v[2] - md[2]};
    double svec[3];
    for (int a = 0; a < 3; ++a) svec[a] = adj[3 * a] * d[0] + adj[3 * a + 1] * d[1] + adj[3 * a + 2] * d[2];
    const double quad = Q[0][0] * d[0] * d[0] + Q[1][1] * d[1] * d[1] + Q[2][2] * d[2] * d[2] +
                        2.0 * (Q[0][1] * d[0] * d[1] + Q[0][2] * d[0] * d[2] + Q[1][2] * d[1] * d[2]);
    const double w = exp(-0.5 * quad) * w_norm;
    const bool cap_open = opacity * w < vp.alpha_max;
    const double cw[3] = {mp[0] + svec[0] - vp.pos[0], mp[1] + svec[1] - vp.pos[1],
                          mp[2] + svec[2] - vp.pos[2]};
    double t[3];
    for (int a = 0; a < 3; ++a) t[a] = R[3 * a] * cw[0] + R[3 * a + 1] * cw[1] + R[3 * a + 2] * cw[2];
    bool clip_open[3];
    for (int c = 0; c < 3; ++c) {
        const double pre = sh_c0 * shc[c] - sh_c1 * v[1] * shc[3 + c] + sh_c1 * v[2] * shc[6 + c] -
                           sh_c1 * v[0] * shc[9 + c] + 0.5;
        clip_open[c] = pre > 0.0 && pre < 1.0;
    }
    const double inv_z = 1.0 / t[2];
    const double ratio_x = t[0] * inv_z, ratio_y = t[1] * inv_z;
    const bool inside_x = fabs(ratio_x) <= vp.lim_x, inside_y = fabs(ratio_y) <= vp.lim_y;
    const double xc = fmin(fmax(ratio_x, -vp.lim_x), vp.lim_x) * t[2];
    const double yc = fmin(fmax(ratio_y, -vp.lim_y), vp.lim_y) * t[2];
    const double j00 = f * inv_z;
    const double j02 = -f * xc * inv_z * inv_z;
    const double j12 = -f * yc * inv_z * inv_z;
    double m3[3][3];   // R sp R^T
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) acc += R[3 * a + p] * sp[3 * p + q] * R[3 * b + q];
            m3[a][b] = acc;
        }
    const double m00 = m3[0][0], m01 = m3[0][1], m02 = m3[0][2], m11 = m3[1][1], m12 = m3[1][2],
                 m22 = m3[2][2];
    const double jm00 = j00 * m00 + j02 * m02, jm01 = j00 * m01 + j02 * m12;
    const double jm02 = j00 * m02 + j02 * m22, jm11 = j00 * m11 + j12 * m12;
    const double jm12 = j00 * m12 + j12 * m22;
    const double cov_a = jm00 * j00 + jm02 * j02 + vp.low_pass;
    const double cov_b = jm01 * j00 + jm02 * j12;
    const double cov_c = jm11 * j00 + jm12 * j12 + vp.low_pass;
    const double inv_det = 1.0 / (cov_a * cov_c - cov_b * cov_b);
    const double ia = cov_c * inv_det, ib = -cov_b * inv_det, ic = cov_a * inv_det;

    // --- reverse sweep ------------------------------------------------------
    const double g_u = gs[0], g_v = gs[1], g_ia = gs[2], g_ib = gs[3], g_ic = gs[4];
    const double g_col[3] = {gs[5], gs[6], gs[7]};
    const double g_alpha = gs[8];
    const double g_cov_a = -(ia * ia * g_ia + ia * ib * g_ib + ib * ib * g_ic);
    const double g_cov_b = -(2.0 * ia * ib * g_ia + (ia * ic + ib * ib) * g_ib + 2.0 * ib * ic * g_ic);
    const double g_cov_c = -(ib * ib * g_ia + ib * ic * g_ib + ic * ic * g_ic);
    const double g_jm00 = g_cov_a * j00, g_jm01 = g_cov_b * j00;
    const double g_jm02 = g_cov_a * j02 + g_cov_b * j12;
    const double g_jm11 = g_cov_c * j00, g_jm12 = g_cov_c * j12;
    const double g_j00 = g_cov_a * jm00 + g_cov_b * jm01 + g_cov_c * jm11 + g_jm00 * m00 + g_jm01 * m01 +
                         g_jm02 * m02 + g_jm11 * m11 + g_jm12 * m12;
    const double g_j02 = g_cov_a * jm02 + g_jm00 * m02 + g_jm01 * m12 + g_jm02 * m22;
    const double g_j12 = g_cov_b * jm02 + g_cov_c * jm12 + g_jm11 * m12 + g_jm12 * m22;
    double g_m3[3][3] = {{g_jm00 * j00, g_jm01 * j00, g_jm00 * j02 + g_jm02 * j00},
                         {0.0, g_jm11 * j00, g_jm01 * j02 + g_jm11 * j12 + g_jm12 * j00},
                         {0.0, 0.0, g_jm02 * j02 + g_jm12 * j12}};
    double g_sp[3][3];   // R^T g_m3 R
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) acc += R[3 * p + a] * g_m3[p][q] * R[3 * q + b];
            g_sp[a][b] = acc;
        }
    double g_tx = g_u * (f * inv_z);
    double g_ty = g_v * (f * inv_z);
    double g_tz = -(g_u * t[0] + g_v * t[1]) * f * inv_z * inv_z;
    g_tz -= g_j00 * f * inv_z * inv_z;
    const double g_xc = -g_j02 * f * inv_z * inv_z;
    const double g_yc = -g_j12 * f * inv_z * inv_z;
    g_tz += 2.0 * f * inv_z * inv_z * inv_z * (g_j02 * xc + g_j12 * yc);
    if (inside_x) g_tx += g_xc;
    else g_tz += g_xc * (ratio_x > 0.0 ? 1.0 : (ratio_x < 0.0 ? -1.0 : 0.0)) * vp.lim_x;
    if (inside_y) g_ty += g_yc;
    else g_tz += g_yc * (ratio_y > 0.0 ? 1.0 : (ratio_y < 0.0 ? -1.0 : 0.0)) * vp.lim_y;
    const double g_t[3] = {g_tx, g_ty, g_tz};
    double g_madj[3];
    for (int k = 0; k < 3; ++k) g_madj[k] = R[k] * g_t[0] + R[3 + k] * g_t[1] + R[6 + k] * g_t[2];

    double g_rgb[3], g_shv[12];
    for (int c = 0; c < 3; ++c) g_rgb[c] = clip_open[c] ? g_col[c] : 0.0;
    for (int c = 0; c < 3; ++c) {
        g_shv[c] = sh_c0 * g_rgb[c];
        g_shv[3 + c] = -sh_c1 * v[1] * g_rgb[c];
        g_shv[6 + c] = sh_c1 * v[2] * g_rgb[c];
        g_shv[9 + c] = -sh_c1 * v[0] * g_rgb[c];
    }
    double g_v3[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < 3; ++c) {
        g_v3[0] += shc[9 + c] * g_rgb[c];
        g_v3[1] += shc[3 + c] * g_rgb[c];
        g_v3[2] += shc[6 + c] * g_rgb[c];
    }
    g_v3[0] *= -sh_c1;
    g_v3[1] *= -sh_c1;
    g_v3[2] *= sh_c1;

    const double g_ap = cap_open ? g_alpha : 0.0;
    const double g_opacity_raw = g_ap * w * opacity * (1.0 - opacity);
    const double g_w = g_ap * opacity;
    const double g_quad = -0.5 * g_w * w;
    double qd[3], g_d[3], g_q[3][3], g_a[3][3];
    for (int a = 0; a < 3; ++a) qd[a] = Q[a][0] * d[0] + Q[a][1] * d[1] + Q[a][2] * d[2];
    for (int a = 0; a < 3; ++a) g_d[a] = 2.0 * g_quad * qd[a];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            g_q[a][b] = g_quad * d[a] * d[b];
            g_a[a][b] = g_madj[a] * d[b];
        }
    for (int j = 0; j < 3; ++j)
        g_d[j] += adj[j] * g_madj[0] + adj[3 + j] * g_madj[1] + adj[6 + j] * g_madj[2];

    // Sigma_pd and the Cholesky factor L (same construction as k_prepare)
    double L[6][6];
    for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b) L[a][b] = 0.0;
    const double scale[6] = {sc.ss[0], sc.ss[1], sc.ss[2], sc.ds, sc.ds, sc.ds};
    for (int k = 0; k < 6; ++k) L[k][k] = scale[k] * exp(raw[k]);
#pragma unroll
    for (int k = 0; k < 15; ++k) L[tril_i(k)][tril_j(k)] = tanh(raw[6 + k]);
    double pd[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int k = 0; k < 6; ++k) acc += L[a][k] * L[3 + b][k];
            pd[a][b] = acc;
        }
    double g_t4[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g_t4[a][b] = -g_sp[a][b];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k)
            g_a[a][k] += g_t4[a][0] * pd[0][k] + g_t4[a][1] * pd[1][k] + g_t4[a][2] * pd[2][k];
    double g_pd[3][3];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) {
            g_pd[a][k] = g_t4[0][a] * adj[k] + g_t4[1][a] * adj[3 + k] + g_t4[2][a] * adj[6 + k];
            g_pd[a][k] += g_a[a][0] * Q[k][0] + g_a[a][1] * Q[k][1] + g_a[a][2] * Q[k][2];
        }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            g_q[a][b] += pd[0][a] * g_a[0][b] + pd[1][a] * g_a[1][b] + pd[2][a] * g_a[2][b];
    double g_sdd[3][3], tmp[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) tmp[a][b] = Q[a][0] * g_q[0][b] + Q[a][1] * g_q[1][b] + Q[a][2] * g_q[2][b];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            g_sdd[a][b] = -(tmp[a][0] * Q[0][b] + tmp[a][1] * Q[1][b] + tmp[a][2] * Q[2][b]);
    if (sc.w_mode == 1)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) g_sdd[a][b] += (-0.5 * g_w * w) * Q[a][b];

    double G[6][6];   // g_sigma + g_sigma^T
    for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b) G[a][b] = 0.0;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            G[a][b] += g_sp[a][b];
            G[b][a] += g_sp[a][b];
            G[a][3 + b] += g_pd[a][b];
            G[3 + b][a] += g_pd[a][b];
            G[3 + a][3 + b] += g_sdd[a][b];
            G[3 + b][3 + a] += g_sdd[a][b];
        }
    double g_raw[21];
    for (int k = 0; k < 6; ++k) {
        double gl = 0.0;
        for (int p = 0; p < 6; ++p) gl += G[k][p] * L[p][k];
        g_raw[k] = gl * L[k][k];
    }
#pragma unroll
    for (int k = 0; k < 15; ++k) {
        const int a = tril_i(k), b = tril_j(k);
        double gl = 0.0;
        for (int p = 0; p < 6; ++p) gl += G[a][p] * L[p][b];
        const double off = L[a][b];
        g_raw[6 + k] = gl * (1.0 - off * off);
    }
    for (int k = 0; k < 3; ++k) g_v3[k] += g_d[k];
    const double vdot = v[0] * g_v3[0] + v[1] * g_v3[1] + v[2] * g_v3[2];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        go[k] = g_madj[k] + (g_v3[k] - v[k] * vdot) * inv_dist;
        go[3 + k] = -g_d[k];
    }
#pragma unroll
    for (int k = 0; k < 21; ++k) go[6 + k] = g_raw[k];
#pragma unroll
    for (int k = 0; k < 12; ++k) go[27 + k] = g_shv[k];
    go[39] = g_opacity_raw;
}

// One thread per scene row, 128 consecutive rows per CTA: the rows' AoS
// inputs (cov_raw, 21 doubles; the splat's screen-space gradient, 9) are
// staged through shared memory with coalesced loads and the 40 outputs leave
// the same way, so every global access is a contiguous block of the CTA's
// rows (per-thread strided rows cost 4x the L1 sectors).  Rows the view did
// not draw get exact zeros (no memset of the gradient arrays).
constexpr int kRowsIn = 30;
__global__ void __launch_bounds__(128, G6R_ROWS_MINB)
k_backward_rows(ViewParams vp, BwdScene sc, g6r_scene scene, int64_t *counters,
                const uint8_t *__restrict__ drawn, const double *__restrict__ gsplat, BwdOut out,
                double sh_c0, double sh_c1) {
    __shared__ double s_io[128 * kRowsIn];
    const int64_t n = scene.n;
    const int64_t i0 = (int64_t)blockIdx.x * 128;
    const int rows = n - i0 < 128 ? (int)(n - i0) : 128;
    const int t = threadIdx.x;
    for (int k = t; k < rows * 21; k += 128) s_io[(k / 21) * kRowsIn + k % 21] = sc.cov_raw[i0 * 21 + k];
    for (int k = t; k < rows * 9; k += 128) s_io[(k / 9) * kRowsIn + 21 + k % 9] = gsplat[i0 * 9 + k];
    __syncthreads();
    double go[kGradOut];
#pragma unroll
    for (int k = 0; k < kGradOut; ++k) go[k] = 0.0;
    if (t < rows && drawn[i0 + t])
        chain_row(vp, sc, reinterpret_cast<const double2 *>(scene.records), n, i0 + t,
                  s_io + t * kRowsIn, s_io + t * kRowsIn + 21, sh_c0, sh_c1, go);
    // non-finite check of the row's outputs: the largest exponent field,
    // all-ones only for inf / nan
    unsigned ex = 0;
#pragma unroll
    for (int k = 0; k < kGradOut; ++k) ex = max(ex, (unsigned)__double2hiint(go[k]) & 0x7ff00000u);
    if (ex == 0x7ff00000u) counters[G6R_CNT_GRAD_NONFINITE] = 1;
    __syncthreads();   // inputs consumed: s_io stages the outputs, one array at a time
#define G6R_PUT_ROWS(dst, off, w)                                                   \
    {                                                                               \
        _Pragma("unroll") for (int k = 0; k < (w); ++k) s_io[t * (w) + k] = go[(off) + k]; \
        __syncthreads();                                                            \
        for (int k = t; k < rows * (w); k += 128) (dst)[i0 * (w) + k] = s_io[k];    \
        __syncthreads();                                                            \
    }
    G6R_PUT_ROWS(out.g_cov_raw, 6, 21)
    G6R_PUT_ROWS(out.g_sh, 27, 12)
    G6R_PUT_ROWS(out.g_mu_p, 0, 3)
    G6R_PUT_ROWS(out.g_mu_d, 3, 3)
#undef G6R_PUT_ROWS
    if (t < rows) out.g_opacity_raw[i0 + t] = go[39];
}

static const double kShC0b = 0.28209479177387814;
static const double kShC1b = 0.4886025119029199;

int launch_backward(const ViewParams &vp, const g6r_scene &scene, const Workspace &ws,
                    int64_t *counters, const double *final_t, const int32_t *last,
                    const double *grad_image, const int64_t *gids, uint8_t *drawn, double *egrad,
                    double *gsplat,
                    const double *mu_p, const double *mu_d, const double *cov_raw, const double *sh,
                    const double *ss, double ds, int w_mode, double *g_mu_p, double *g_mu_d,
                    double *g_cov_raw, double *g_sh, double *g_opacity_raw, cudaStream_t st) {
    if (vp.tile_size != 16) return G6R_EINVAL;
    const int64_t n = scene.n;
    cudaMemsetAsync(counters + G6R_CNT_GRAD_NONFINITE, 0, sizeof(int64_t), st);
    if (n == 0) return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
    k_zero_rows<<<148 * 4, 256, 0, st>>>(counters, ws.entry_capacity, egrad, n, drawn);
    k_composite_bwd<<<vp.tiles_x * vp.tiles_y * 2, 128, 0, st>>>(
        vp, static_cast<const PayloadF64 *>(ws.payload), ws.vals[0], ws.vals[1], ws.internal,
        ws.tile_starts, final_t, last, grad_image, ws.splat_rect, egrad, ws.entry_capacity);
    trace_mark("composite_bwd", st);
    const unsigned grid = (unsigned)ceil_div(n, 128);
    k_splat_grad_sum<<<grid, 128, 0, st>>>(n, ws.splat_rect, counters, egrad, ws.entry_capacity, gids,
                                           gsplat, drawn);
    trace_mark("splat_grad_sum", st);
    BwdScene sc{mu_p, mu_d, cov_raw, sh, {ss[0], ss[1], ss[2]}, ds, w_mode};
    BwdOut out{g_mu_p, g_mu_d, g_cov_raw, g_sh, g_opacity_raw};
    k_backward_rows<<<grid, 128, 0, st>>>(vp, sc, scene, counters, drawn, gsplat, out, kShC0b, kShC1b);
    trace_mark("backward_rows", st);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
