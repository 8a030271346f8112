// g6r_train.cu -- photometric loss with its image gradient, and Adam, on device
// (the fine-tune loop of diffrender.py:548-585 around the render path).
//
// Replaces diffrender.py:117-138 (_loss_parts: L1 + (1 - MS-SSIM)),
// _ssim.py:23-201 (11x11 sigma-1.5 valid windows, 2x2 pooling pyramid,
// per-scale contrast-structure means, analytic gradient) and
// diffrender.py:481-509 (adam_step).  Reductions are deterministic (fixed
// block partials, then one ordered final sum); Adam follows the reference's
// operation order element for element.
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <vector>
#include <cmath>
#include <vector>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

constexpr int kWin = 11;
constexpr int kRedBlocks = 256;   // fixed partial count for deterministic sums
__constant__ double c_win[kWin];

// Gaussian window (_ssim.py:25-30): exp(-x^2 / (2 s^2)) normalised, s = 1.5.
static void window_host(double *w) {
    double s = 0.0;
    for (int k = 0; k < kWin; ++k) {
        const double x = k - (kWin - 1) / 2.0;
        w[k] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
        s += w[k];
    }
    for (int k = 0; k < kWin; ++k) w[k] /= s;
}

// The three colour channels of the MS-SSIM term are independent: every
// per-channel kernel below takes its channel from blockIdx.y (blockIdx.z for
// the correlation) and its planes `cs` doubles apart, so one launch covers the
// channels with each channel's arithmetic unchanged.

// planar channel c of the interleaved (H, W, 4) prediction and (H, W, tc) target
__global__ void k_extract(const double *__restrict__ pred, const double *__restrict__ tgt, int tc,
                          int64_t hw, double *__restrict__ x, double *__restrict__ y, int64_t cs) {
    const int c = blockIdx.y;
    x += c * cs;
    y += c * cs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = pred[i * 4 + c];
        y[i] = tgt[i * tc + c];
    }
}

// 5 statistic planes x, y, x*x, y*y, x*y
__global__ void k_products(const double *__restrict__ x, const double *__restrict__ y, int64_t hw,
                           double *__restrict__ out, int64_t cs) {
    x += blockIdx.y * cs;
    y += blockIdx.y * cs;
    out += blockIdx.y * cs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = x[i], b = y[i];
        out[i] = a;
        out[hw + i] = b;
        out[2 * hw + i] = a * a;
        out[3 * hw + i] = b * b;
        out[4 * hw + i] = a * b;
    }
}

// 1-D correlation with the window along one axis of `planes` (h, w) planes.
// valid: out length n - 10; full: n + 10 (zero padding, the adjoint).
// grid (column blocks of 128, row blocks of kCorrRows, channels x planes).
// The CTA stages the input window of its output tile through shared memory
// with coalesced loads (zeros outside the image), then every thread sums its
// column's taps for kCorrRows output rows from shared memory: each input is
// read from L2 about once instead of once per tap.  Same taps, same order
// (k ascending), out-of-image taps skipped as before: identical bits.
constexpr int kCorrCols = 128, kCorrRows = 16;
template <int kAxis>
__global__ void __launch_bounds__(kCorrCols)
k_corr1d(const double *__restrict__ in, double *__restrict__ out, int planes, int h, int w, int full,
         int64_t cs) {
    constexpr int SH = kAxis == 0 ? kCorrRows + kWin - 1 : kCorrRows;   // staged rows
    constexpr int SW = kAxis == 0 ? kCorrCols : kCorrCols + kWin - 1;   // staged columns
    __shared__ double s_in[SH * SW];
    const int oh = kAxis == 0 ? (full ? h + kWin - 1 : h - kWin + 1) : h;
    const int ow = kAxis == 1 ? (full ? w + kWin - 1 : w - kWin + 1) : w;
    const int shift = full ? kWin - 1 : 0;
    const int c = blockIdx.z / planes, p = blockIdx.z - c * planes;
    const double *src = in + c * cs + (int64_t)p * h * w;
    double *dst = out + c * cs + (int64_t)p * oh * ow;
    const int j0 = blockIdx.x * kCorrCols, i0 = blockIdx.y * kCorrRows;
    // input window origin: (i0 - shift, j0) vertically, (i0, j0 - shift) horizontally
    const int ri = kAxis == 0 ? i0 - shift : i0, rj = kAxis == 1 ? j0 - shift : j0;
    for (int q = threadIdx.x; q < SH * SW; q += kCorrCols) {
        const int a = q / SW, b = q - a * SW;
        const int ii = ri + a, jj = rj + b;
        s_in[q] = (ii >= 0 && ii < h && jj >= 0 && jj < w) ? src[(int64_t)ii * w + jj] : 0.0;
    }
    __syncthreads();
    const int j = j0 + threadIdx.x;
    if (j >= ow) return;
    for (int r = 0; r < kCorrRows; ++r) {
        const int i = i0 + r;
        if (i >= oh) break;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const int ii = kAxis == 0 ? i + k - shift : i;
            const int jj = kAxis == 1 ? j + k - shift : j;
            if (ii >= 0 && ii < h && jj >= 0 && jj < w)
                s += c_win[k] * (kAxis == 0 ? s_in[(r + k) * SW + threadIdx.x]
                                            : s_in[r * SW + threadIdx.x + k]);
        }
        dst[(int64_t)i * ow + j] = s;
    }
}

static dim3 corr_grid(int planes, int h, int w, int axis, int full) {
    const int oh = axis == 0 ? (full ? h + kWin - 1 : h - kWin + 1) : h;
    const int ow = axis == 1 ? (full ? w + kWin - 1 : w - kWin + 1) : w;
    return dim3((unsigned)((ow + kCorrCols - 1) / kCorrCols),
                (unsigned)std::max((oh + kCorrRows - 1) / kCorrRows, 1), (unsigned)(3 * planes));
}

// SSIM window maps (_ssim.py:66-84) from the 5 correlated statistics
__global__ void k_ssim_maps(const double *__restrict__ st, int64_t n, double *__restrict__ maps,
                            int64_t cs) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    st += blockIdx.y * cs;
    maps += blockIdx.y * cs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double ux = st[i], uy = st[n + i], exx = st[2 * n + i], eyy = st[3 * n + i], exy = st[4 * n + i];
        const double sxx = exx - ux * ux, syy = eyy - uy * uy, sxy = exy - ux * uy;
        const double b1 = ux * ux + uy * uy + C1;
        const double b2 = sxx + syy + C2;
        maps[i] = ux;
        maps[n + i] = uy;
        maps[2 * n + i] = b1;
        maps[3 * n + i] = b2;
        maps[4 * n + i] = (2.0 * ux * uy + C1) / b1;   // l
        maps[5 * n + i] = (2.0 * sxy + C2) / b2;       // cs
    }
}

// deterministic partial sums: block b sums a fixed strided subset
// (channel blockIdx.y: a, b `cs` doubles apart, partials kRedBlocks apart)
__global__ void k_partials(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                           double *__restrict__ part, int64_t cs) {
    __shared__ double s[256];
    a += blockIdx.y * cs;
    if (b) b += blockIdx.y * cs;
    part += blockIdx.y * gridDim.x;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += b ? a[i] * b[i] : a[i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

// ordered final sum of block b's n partials into out[b * ostride]: the
// partials are staged in shared memory by the whole block (one memory round
// trip instead of n dependent-latency loads), then summed by one thread in
// index order
__global__ void k_sum_partials(const double *__restrict__ part, int n, double *__restrict__ out,
                               int ostride) {
    __shared__ double s[kRedBlocks];
    part += (int64_t)blockIdx.x * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = part[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += s[i];
        out[(int64_t)blockIdx.x * ostride] = acc;
    }
}

// per-window gradients of SsimParts.backward (_ssim.py:86-98) for constant
// per-window upstream gradients g_lcs, g_cs
// (g_scale of channel c at g_scale[c * gstride])
__global__ void k_ssim_bwd_maps(const double *__restrict__ maps, int64_t n, const double *g_scale,
                                int gstride, int last, double *__restrict__ gm, int64_t cs) {
    maps += blockIdx.y * cs;
    gm += blockIdx.y * cs;
    g_scale += blockIdx.y * gstride;
    // per-window upstream gradient of this scale, computed on the device
    const double g_lcs = last ? *g_scale : 0.0, g_cs = last ? 0.0 : *g_scale;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double ux = maps[i], uy = maps[n + i], b1 = maps[2 * n + i], b2 = maps[3 * n + i];
        const double l = maps[4 * n + i], cs = maps[5 * n + i];
        const double g_l = g_lcs * cs;
        const double g_cst = g_lcs * l + g_cs;
        gm[i] = g_l * 2.0 * (uy - l * ux) / b1 + g_cst * 2.0 * (cs * ux - uy) / b2;   // g_ux
        gm[n + i] = -g_cst * cs / b2;                                                  // g_exx
        gm[2 * n + i] = g_cst * 2.0 / b2;                                              // g_exy
    }
}

// g += adj(g_ux) + 2 x adj(g_exx) + y adj(g_exy)
__global__ void k_ssim_bwd_combine(const double *__restrict__ adj, const double *__restrict__ x,
                                   const double *__restrict__ y, int64_t hw, double *__restrict__ g,
                                   int64_t cs) {
    adj += blockIdx.y * cs;
    x += blockIdx.y * cs;
    y += blockIdx.y * cs;
    g += blockIdx.y * cs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x)
        g[i] += adj[i] + 2.0 * x[i] * adj[hw + i] + y[i] * adj[2 * hw + i];
}

// 2x2 average pooling (_ssim.py:47-51) of x and y, and its adjoint (:54-62)
__global__ void k_pool2(const double *__restrict__ x, const double *__restrict__ y, int h, int w,
                        double *__restrict__ x2, double *__restrict__ y2, int64_t cs) {
    const int h2 = h / 2, w2 = w / 2;
    x += blockIdx.y * cs;
    y += blockIdx.y * cs;
    x2 += blockIdx.y * cs;
    y2 += blockIdx.y * cs;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)h2 * w2;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(q / w2), j = (int)(q % w2);
        const int64_t o = (int64_t)(2 * i) * w + 2 * j;
        x2[q] = 0.25 * (x[o] + x[o + w] + x[o + 1] + x[o + w + 1]);
        y2[q] = 0.25 * (y[o] + y[o + w] + y[o + 1] + y[o + w + 1]);
    }
}

__global__ void k_pool2_adjoint(const double *__restrict__ g2, int h, int w, double *__restrict__ out,
                                int64_t cs) {
    const int h2 = h / 2, w2 = w / 2;
    g2 += blockIdx.y * cs;
    out += blockIdx.y * cs;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)h * w;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(q / w), j = (int)(q % w);
        out[q] = (i < 2 * h2 && j < 2 * w2) ? 0.25 * g2[(int64_t)(i / 2) * w2 + j / 2] : 0.0;
    }
}

// L1 part: diff statistics and grad = l1_w * sign(diff) / size on RGB
__global__ void k_l1(const double *__restrict__ pred, const double *__restrict__ tgt, int tc,
                     int64_t hw, double scale, double *__restrict__ grad, double *__restrict__ absdiff) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < hw * 3; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = q / 3;
        const int c = (int)(q % 3);
        const double d = pred[p * 4 + c] - tgt[p * tc + c];
        absdiff[q] = fabs(d);
        grad[p * 4 + c] = scale * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0));
        if (c == 0) grad[p * 4 + 3] = 0.0;
    }
}

__global__ void k_axpy_channel(const double *__restrict__ g, int64_t hw, double alpha,
                               double *__restrict__ grad, int64_t cs) {
    const int c = blockIdx.y;
    g += c * cs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x)
        grad[i * 4 + c] += alpha * g[i];
}

// bias-corrected Adam (diffrender.py:493-508), the reference's operation order
__device__ __forceinline__ void adam_one(double &p, double g, double &m, double &v, double lr,
                                         double bias1, double bias2) {
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    double mi = m * b1;
    mi = mi + (1.0 - b1) * g;
    double vi = v * b2;
    vi = vi + (1.0 - b2) * (g * g);
    m = mi;
    v = vi;
    p = p - lr * (mi / bias1) / (sqrt(vi / bias2) + eps);
}

// 16-byte accesses (pairs of parameters) when the four arrays are 16-byte
// aligned; the per-element operations are unchanged
__global__ void k_adam(int64_t n, double *__restrict__ p, const double *__restrict__ g,
                       double *__restrict__ m, double *__restrict__ v, double lr, double bias1,
                       double bias2) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                       reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
    int64_t done = 0;
    if (vec) {
        const int64_t n2 = n / 2;
        double2 *p2 = reinterpret_cast<double2 *>(p), *m2 = reinterpret_cast<double2 *>(m),
                *v2 = reinterpret_cast<double2 *>(v);
        const double2 *g2 = reinterpret_cast<const double2 *>(g);
        for (int64_t i = t0; i < n2; i += stride) {
            double2 pp = p2[i], mm = m2[i], vv = v2[i];
            const double2 gg = g2[i];
            adam_one(pp.x, gg.x, mm.x, vv.x, lr, bias1, bias2);
            adam_one(pp.y, gg.y, mm.y, vv.y, lr, bias1, bias2);
            m2[i] = mm;
            v2[i] = vv;
            p2[i] = pp;
        }
        done = 2 * n2;
    }
    for (int64_t i = done + t0; i < n; i += stride) {
        double pp = p[i], mm = m[i], vv = v[i];
        adam_one(pp, g[i], mm, vv, lr, bias1, bias2);
        m[i] = mm;
        v[i] = vv;
        p[i] = pp;
    }
}

__global__ void k_nonfinite(int64_t n, const double *__restrict__ x, int32_t *__restrict__ flag) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

static unsigned grid_for(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8));
}

// --- host orchestration -------------------------------------------------------

// x .. g: channel 0's planes; channel c's are c * cstride bytes further on
struct LossLayout {
    size_t x[5], y[5], maps[5], stats, tmp, gm, adj, g, cstride, part, scal, absd, in_pred, in_tgt,
        out_grad, total;
};

static inline size_t al(size_t v) { return (v + 255) & ~size_t(255); }

static LossLayout loss_layout(int h, int w, int scales) {
    LossLayout L{};
    size_t o = 0;
    int hh = h, ww = w;
    for (int j = 0; j < scales; ++j) {
        const size_t hw = (size_t)hh * ww;
        const size_t nv = (size_t)std::max(hh - kWin + 1, 0) * std::max(ww - kWin + 1, 0);
        L.x[j] = o;
        o = al(o + hw * 8);
        L.y[j] = o;
        o = al(o + hw * 8);
        L.maps[j] = o;
        o = al(o + 6 * nv * 8);
        hh /= 2;
        ww /= 2;
    }
    const size_t hw = (size_t)h * w;
    L.stats = o;
    o = al(o + 5 * hw * 8);
    L.tmp = o;
    o = al(o + 5 * hw * 8);
    L.gm = o;
    o = al(o + 3 * hw * 8);
    L.adj = o;
    o = al(o + 3 * hw * 8);
    L.g = o;
    o = al(o + 2 * hw * 8);
    L.cstride = o;
    o *= 3;
    L.part = o;
    o = al(o + 3 * kRedBlocks * 8);
    L.scal = o;
    o = al(o + 64 * 8);
    L.absd = o;
    o = al(o + 3 * hw * 8);
    // fixed-address copies of the call's pred / target / gradient, so the
    // captured graph of the loss can be replayed for any caller buffers
    L.in_pred = o;
    o = al(o + 4 * hw * 8);
    L.in_tgt = o;
    o = al(o + 4 * hw * 8);
    L.out_grad = o;
    o = al(o + 4 * hw * 8);
    L.total = o;
    return L;
}

size_t loss_workspace_bytes(int h, int w) { return loss_layout(h, w, 5).total; }

// sum of a*b (or a) over n doubles into *out (device), deterministic; for
// nch channels (a, b `cs` doubles apart) into out[c * ostride]
static void dsum(const double *a, const double *b, int64_t n, int nch, int64_t cs, double *part,
                 double *out, int ostride, cudaStream_t st) {
    k_partials<<<dim3(kRedBlocks, nch), 256, 0, st>>>(a, b, n, part, cs);
    k_sum_partials<<<nch, 256, 0, st>>>(part, kRedBlocks, out, ostride);
}

// Scalar slots of the loss workspace (device doubles).
constexpr int kSlotL1 = 0, kSlotParts = 1;   // l1 sum; total, l1, ssim_loss
constexpr int kSlotChan = 8, kChanStride = 16;   // per channel: sums[5], value, g[5]

struct ScaleWeights {
    double w[5], count[5];
};

// MS-SSIM value and per-scale window gradients of one channel (_ssim.py:163-198):
// terms = means (clamped at 0 for the multi-scale product), value = prod(terms^w),
// g[j] = value * w_j / terms_j / count_j (0 where the reference skips the scale).
__global__ void k_msssim_scalars(double *chan, int ns, ScaleWeights sw) {   // block c: channel c
    if (threadIdx.x != 0) return;
    chan += blockIdx.x * kChanStride;
    double terms[5];
    for (int j = 0; j < ns; ++j) terms[j] = chan[j] / sw.count[j];
    double *g = chan + 6;
    if (ns == 1) {
        chan[5] = terms[0];
        g[0] = 1.0 / sw.count[0];
        return;
    }
    double value = 1.0;
    for (int j = 0; j < ns; ++j) {
        terms[j] = terms[j] > 0.0 ? terms[j] : 0.0;
        value *= pow(terms[j], sw.w[j]);
    }
    chan[5] = value;
    for (int j = 0; j < ns; ++j)
        g[j] = (value > 0.0 && terms[j] > 0.0) ? value * sw.w[j] / terms[j] / sw.count[j] : 0.0;
}

__global__ void k_loss_parts(double *scal, int use_ssim, double lambda_l1, double lambda_ssim,
                             double n_l1) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double l1 = scal[kSlotL1] / n_l1;
    double ssim_value = 0.0;
    if (use_ssim) {
        double total = 0.0;
        for (int c = 0; c < 3; ++c) total += scal[kSlotChan + c * kChanStride + 5];
        ssim_value = total / 3.0;
    }
    const double ssim_loss = use_ssim ? 1.0 - ssim_value : 0.0;
    scal[kSlotParts] = lambda_l1 * l1 + lambda_ssim * ssim_loss;
    scal[kSlotParts + 1] = l1;
    scal[kSlotParts + 2] = ssim_loss;
}

// Every kernel of one loss evaluation, asynchronous on st (graph-capturable);
// the scalar parts end in scal[kSlotParts..] on the device.
static void loss_launch(const double *pred, const double *tgt, int tc, int h, int w, double lambda_l1,
                        double lambda_ssim, int scales, const double *weights_in, void *ws,
                        double *grad, cudaStream_t st) {
    char *base = static_cast<char *>(ws);
    const int64_t hw = (int64_t)h * w;
    const LossLayout L = loss_layout(h, w, 5);
    double *part = reinterpret_cast<double *>(base + L.part);
    double *scal = reinterpret_cast<double *>(base + L.scal);
    // L1 (diffrender.py:126-129)
    double *absd = reinterpret_cast<double *>(base + L.absd);
    k_l1<<<grid_for(hw * 3), 256, 0, st>>>(pred, tgt, tc, hw, lambda_l1 / (double)(hw * 3), grad, absd);
    dsum(absd, nullptr, hw * 3, 1, 0, part, scal + kSlotL1, 0, st);
    if (lambda_ssim > 0.0) {
        // effective_scales (_ssim.py:116-120)
        const int ns = std::min(h, w) < (1 << (scales - 1)) * kWin ? 1 : scales;
        ScaleWeights sw{};
        double wsum = 0.0;
        for (int j = 0; j < ns; ++j) wsum += weights_in[j];
        for (int j = 0; j < ns; ++j) sw.w[j] = weights_in[j] / wsum;
        int hs[5], wsz[5];
        hs[0] = h;
        wsz[0] = w;
        for (int j = 1; j < ns; ++j) {
            hs[j] = hs[j - 1] / 2;
            wsz[j] = wsz[j - 1] / 2;
        }
        for (int j = 0; j < ns; ++j)
            sw.count[j] = (double)((int64_t)(hs[j] - kWin + 1) * (wsz[j] - kWin + 1));
        // all three channels per launch (grid y / z), channel c's planes cs doubles on
        const int64_t cs = (int64_t)(L.cstride / 8);
        double *chan = scal + kSlotChan;   // channel c's scalars kChanStride further on
        double *xs[5], *ys[5], *mp[5];
        for (int j = 0; j < ns; ++j) {
            xs[j] = reinterpret_cast<double *>(base + L.x[j]);
            ys[j] = reinterpret_cast<double *>(base + L.y[j]);
            mp[j] = reinterpret_cast<double *>(base + L.maps[j]);
        }
        double *stats = reinterpret_cast<double *>(base + L.stats);
        double *tmp = reinterpret_cast<double *>(base + L.tmp);
        k_extract<<<dim3(grid_for(hw), 3), 256, 0, st>>>(pred, tgt, tc, hw, xs[0], ys[0], cs);
        for (int j = 0; j < ns; ++j) {
            const int hj = hs[j], wj = wsz[j];
            const int64_t hwj = (int64_t)hj * wj;
            const int hv = hj - kWin + 1, wv = wj - kWin + 1;
            const int64_t nv = (int64_t)hv * wv;
            k_products<<<dim3(grid_for(hwj), 3), 256, 0, st>>>(xs[j], ys[j], hwj, stats, cs);
            k_corr1d<0><<<corr_grid(5, hj, wj, 0, 0), kCorrCols, 0, st>>>(stats, tmp, 5, hj, wj, 0, cs);
            k_corr1d<1><<<corr_grid(5, hv, wj, 1, 0), kCorrCols, 0, st>>>(tmp, stats, 5, hv, wj, 0, cs);
            k_ssim_maps<<<dim3(grid_for(nv), 3), 256, 0, st>>>(stats, nv, mp[j], cs);
            if (j == ns - 1) dsum(mp[j] + 4 * nv, mp[j] + 5 * nv, nv, 3, cs, part, chan + j, kChanStride, st);
            else dsum(mp[j] + 5 * nv, nullptr, nv, 3, cs, part, chan + j, kChanStride, st);
            if (j + 1 < ns)
                k_pool2<<<dim3(grid_for(hwj / 4 + 1), 3), 256, 0, st>>>(xs[j], ys[j], hj, wj, xs[j + 1],
                                                                       ys[j + 1], cs);
        }
        k_msssim_scalars<<<3, 32, 0, st>>>(chan, ns, sw);
        // backward from the coarsest scale (_ssim.py:175-198)
        double *g = reinterpret_cast<double *>(base + L.g);
        double *g2 = g + hw;
        cudaMemset2DAsync(g, L.cstride, 0, (size_t)hs[ns - 1] * wsz[ns - 1] * 8, 3, st);
        double *gm = reinterpret_cast<double *>(base + L.gm);
        double *adj = reinterpret_cast<double *>(base + L.adj);
        for (int j = ns - 1; j >= 0; --j) {
            const int hj = hs[j], wj = wsz[j];
            const int64_t hwj = (int64_t)hj * wj;
            const int hv = hj - kWin + 1, wv = wj - kWin + 1;
            const int64_t nv = (int64_t)hv * wv;
            if (j < ns - 1) {   // upsample the coarser gradient into this level
                k_pool2_adjoint<<<dim3(grid_for(hwj), 3), 256, 0, st>>>(g, hj, wj, g2, cs);
                std::swap(g, g2);
            }
            k_ssim_bwd_maps<<<dim3(grid_for(nv), 3), 256, 0, st>>>(mp[j], nv, chan + 6 + j, kChanStride,
                                                                  j == ns - 1, gm, cs);
            k_corr1d<0><<<corr_grid(3, hv, wv, 0, 1), kCorrCols, 0, st>>>(gm, tmp, 3, hv, wv, 1, cs);
            k_corr1d<1><<<corr_grid(3, hj, wv, 1, 1), kCorrCols, 0, st>>>(tmp, adj, 3, hj, wv, 1, cs);
            k_ssim_bwd_combine<<<dim3(grid_for(hwj), 3), 256, 0, st>>>(adj, xs[j], ys[j], hwj, g, cs);
        }
        // grad_rgb -= lambda_ssim * g_ms, with g_ms averaged over channels
        k_axpy_channel<<<dim3(grid_for(hw), 3), 256, 0, st>>>(g, hw, -lambda_ssim / 3.0, grad, cs);
    }
    k_loss_parts<<<1, 32, 0, st>>>(scal, lambda_ssim > 0.0, lambda_l1, lambda_ssim, (double)(hw * 3));
}

// The ~75 small kernels of one loss evaluation are captured once per
// (device, workspace, image size, channels, weights) into a CUDA graph on a
// private stream and replayed: one launch instead of ~75, same kernels in the
// same order, hence the same bits.  The caller's buffers are copied to / from
// fixed workspace regions around the replay.
struct LossGraph {
    int dev, h, w, tc, scales;
    double l1, ssim, weights[5];
    void *ws;
    cudaStream_t stream;
    cudaEvent_t in, out;
    cudaGraphExec_t exec;
};
static std::vector<LossGraph> g_loss_graphs;
static std::mutex g_loss_mu;
constexpr size_t kMaxLossGraphs = 8;   // bounded: callers that allocate a workspace per call evict

static void destroy_graph(LossGraph &g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.in) cudaEventDestroy(g.in);
    if (g.out) cudaEventDestroy(g.out);
    if (g.stream) cudaStreamDestroy(g.stream);
    g.exec = nullptr;
    g.in = g.out = nullptr;
    g.stream = nullptr;
}

int loss_grad(const double *pred, const double *tgt, int tc, int h, int w, double lambda_l1,
              double lambda_ssim, int scales, const double *weights_in, void *ws, double *grad,
              double *parts, cudaStream_t st) {
    static bool win_set[64] = {};   // __constant__ lives per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return G6R_EINVAL;
    // one caller at a time: the graph cache, the window constants and the
    // replay (every call ends synchronised, so no cached graph is in flight
    // when another call evicts it)
    std::lock_guard<std::mutex> lock(g_loss_mu);
    if (!win_set[dev]) {
        double wv[kWin];
        window_host(wv);
        cudaMemcpyToSymbol(c_win, wv, sizeof wv);
        win_set[dev] = true;
    }
    char *base = static_cast<char *>(ws);
    const int64_t hw = (int64_t)h * w;
    const LossLayout L = loss_layout(h, w, 5);
    double *scal = reinterpret_cast<double *>(base + L.scal);
    double *ipred = reinterpret_cast<double *>(base + L.in_pred);
    double *itgt = reinterpret_cast<double *>(base + L.in_tgt);
    double *ograd = reinterpret_cast<double *>(base + L.out_grad);
    LossGraph *gr = nullptr;
    for (size_t k = 0; k < g_loss_graphs.size(); ++k) {
        const LossGraph &g = g_loss_graphs[k];
        bool same = g.dev == dev && g.h == h && g.w == w && g.tc == tc && g.scales == scales &&
                    g.l1 == lambda_l1 && g.ssim == lambda_ssim && g.ws == ws;
        for (int j = 0; same && j < scales; ++j) same = g.weights[j] == weights_in[j];
        if (same) {   // move to the back (most recently used)
            std::rotate(g_loss_graphs.begin() + k, g_loss_graphs.begin() + k + 1, g_loss_graphs.end());
            gr = &g_loss_graphs.back();
            break;
        }
    }
    if (!gr) {
        if (g_loss_graphs.size() >= kMaxLossGraphs) {   // evict the least recently used
            destroy_graph(g_loss_graphs.front());
            g_loss_graphs.erase(g_loss_graphs.begin());
        }
        LossGraph g{};
        g.dev = dev;
        g.h = h;
        g.w = w;
        g.tc = tc;
        g.scales = scales;
        g.l1 = lambda_l1;
        g.ssim = lambda_ssim;
        for (int j = 0; j < scales; ++j) g.weights[j] = weights_in[j];
        g.ws = ws;
        cudaGraph_t graph = nullptr;
        bool ok = cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreateWithFlags(&g.in, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&g.out, cudaEventDisableTiming) == cudaSuccess &&
                  cudaStreamBeginCapture(g.stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            loss_launch(ipred, itgt, tc, h, w, lambda_l1, lambda_ssim, scales, weights_in, ws, ograd,
                        g.stream);
            ok = cudaStreamEndCapture(g.stream, &graph) == cudaSuccess &&
                 cudaGraphInstantiate(&g.exec, graph, 0) == cudaSuccess;
        }
        if (graph) cudaGraphDestroy(graph);
        if (!ok) {
            destroy_graph(g);
            return G6R_ECUDA;
        }
        g_loss_graphs.push_back(g);
        gr = &g_loss_graphs.back();
    }
    cudaMemcpyAsync(ipred, pred, (size_t)hw * 4 * sizeof(double), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(itgt, tgt, (size_t)hw * tc * sizeof(double), cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(gr->in, st);
    cudaStreamWaitEvent(gr->stream, gr->in, 0);
    cudaGraphLaunch(gr->exec, gr->stream);
    cudaEventRecord(gr->out, gr->stream);
    cudaStreamWaitEvent(st, gr->out, 0);
    cudaMemcpyAsync(grad, ograd, (size_t)hw * 4 * sizeof(double), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(parts, scal + kSlotParts, 3 * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);   // the one read-back of the call
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int adam_step(int64_t n, double *p, const double *g, double *m, double *v, double lr, double bias1,
              double bias2, cudaStream_t st) {
    if (n == 0) return G6R_OK;
    k_adam<<<grid_for(n), 256, 0, st>>>(n, p, g, m, v, lr, bias1, bias2);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int nonfinite(int64_t n, const double *x, int32_t *flag, cudaStream_t st) {
    if (n == 0) return G6R_OK;
    k_nonfinite<<<grid_for(n), 256, 0, st>>>(n, x, flag);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
