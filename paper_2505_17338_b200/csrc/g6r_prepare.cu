// g6r_prepare.cu -- per-scene, view-independent slicing terms on the device.
//
// Replaces raster.py:120-137 prepare_scene -> core.py:255-351
// (cholesky_factor_batch, build_covariance_batch, inv3_batch,
// conditioning_terms) and core.py:54-62 (sigmoid).  One thread per Gaussian;
// the summation orders reproduce numpy's einsum orders on the reference host
// (pinned in SURVEY.md 8a-2 and checked against the oracle in tests).
// Output is the 44-double record of include/g6r.h in 16-byte column packets,
// read by the per-view projection with coalesced 16-byte loads.
#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

__device__ __forceinline__ void put_record(double2 *rec, int64_t n, int64_t i, const double *r44) {
#pragma unroll
    for (int c = 0; c < G6R_REC_COLUMNS; ++c) rec[c * n + i] = make_double2(r44[2 * c], r44[2 * c + 1]);
}

__device__ __forceinline__ double sigmoid_ref(double x) {
    // core.py:54-62: the branch split matters for the rounding
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    const double ex = exp(x);
    return ex / (1.0 + ex);
}

__global__ void __launch_bounds__(kBlock)
k_prepare(int64_t n, const double *__restrict__ mu_p, const double *__restrict__ mu_d,
          const double *__restrict__ cov_raw, const double *__restrict__ sh,
          const double *__restrict__ opacity_raw, const uint8_t *__restrict__ labels,
          double s0, double s1, double s2, double ds, int w_mode, double w_raw_const,
          double2 *__restrict__ rec, uint8_t *__restrict__ flags,
          unsigned long long *__restrict__ label_counts) {
    __shared__ unsigned s_cnt[32];
    if (threadIdx.x < 32) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double *raw = cov_raw + 21 * i;
        double L[6][6];
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int b = 0; b < 6; ++b) L[a][b] = 0.0;
        const double scale[6] = {s0, s1, s2, ds, ds, ds};
#pragma unroll
        for (int d = 0; d < 6; ++d) L[d][d] = scale[d] * exp(raw[d]);
#pragma unroll
        for (int k = 0; k < 15; ++k) L[tril_i(k)][tril_j(k)] = tanh(raw[6 + k]);

        // Sigma[a][b] = ((p0+p2)+p4) + ((p1+p3)+p5), p_j = L[a][j] L[b][j]
        double S[6][6];
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int b = 0; b < 6; ++b) {
                double p[6];
#pragma unroll
                for (int j = 0; j < 6; ++j) p[j] = L[a][j] * L[b][j];
                S[a][b] = ((p[0] + p[2]) + p[4]) + ((p[1] + p[3]) + p[5]);
            }

        // adjugate inverse of the directional block (core.py:275-302)
        const double A = S[3][3], B = S[3][4], C = S[3][5];
        const double D = S[4][3], E = S[4][4], F = S[4][5];
        const double G = S[5][3], H = S[5][4], I = S[5][5];
        const double co00 = E * I - F * H;
        const double co01 = F * G - D * I;
        const double co02 = D * H - E * G;
        const double det = A * co00 + B * co01 + C * co02;
        double P[3][3] = {{co00, C * H - B * I, B * F - C * E},
                          {co01, A * I - C * G, C * D - A * F},
                          {co02, B * G - A * H, A * E - B * D}};
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) P[a][b] = P[a][b] / det;
        // degenerate policy (core.py:331-333)
        const double trace = (A + E) + I;
        const double tcl = (trace > 1e-30 || isnan(trace)) ? trace : 1e-30;   // np.maximum
        const bool degenerate = !isfinite(det) || det <= 1e-30 * pow(tcl, 3.0);
        if (degenerate) {
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) P[a][b] = 0.0;
        }
        // adjust = S_pd P ; sigma' = S_pp - adjust S_pd^T (core.py:334-335)
        double adj[3][3], sp[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                adj[a][b] = (S[a][3] * P[0][b] + S[a][4] * P[1][b]) + S[a][5] * P[2][b];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const double q0 = adj[a][0] * S[b][3];
                const double q1 = adj[a][1] * S[b][4];
                const double q2 = adj[a][2] * S[b][5];
                sp[a][b] = S[a][b] - ((q0 + q2) + q1);
            }
        double w_norm = 1.0;
        if (w_mode == 1) w_norm = degenerate ? 0.0 : w_raw_const / sqrt(det);

        double r44[G6R_REC_DOUBLES];
        r44[0] = mu_p[3 * i];
        r44[1] = mu_p[3 * i + 1];
        r44[2] = mu_p[3 * i + 2];
        r44[3] = mu_d[3 * i];
        r44[4] = mu_d[3 * i + 1];
        r44[5] = mu_d[3 * i + 2];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) r44[6 + 3 * a + b] = adj[a][b];
        r44[15] = P[0][0];
        r44[16] = P[1][1];
        r44[17] = P[2][2];
        r44[18] = P[0][1];
        r44[19] = P[0][2];
        r44[20] = P[1][2];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) r44[21 + 3 * a + b] = sp[a][b];
#pragma unroll
        for (int k = 0; k < 12; ++k) r44[30 + k] = sh[12 * i + k];
        r44[42] = sigmoid_ref(opacity_raw[i]);
        r44[43] = w_norm;
        put_record(rec, n, i, r44);
        const unsigned lab = labels[i] & 15u;
        flags[i] = (uint8_t)(lab | (degenerate ? G6R_FLAG_DEGENERATE : 0u));
        atomicAdd(&s_cnt[lab], 1u);
        if (degenerate) atomicAdd(&s_cnt[16 + lab], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32 && s_cnt[threadIdx.x]) atomicAdd(&label_counts[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(kBlock)
k_pack_records(int64_t n, const double *__restrict__ mu_p, const double *__restrict__ mu_d,
               const double *__restrict__ sh, const double *__restrict__ opacity,
               const double *__restrict__ w_norm, const double *__restrict__ adjust,
               const double *__restrict__ prec, const double *__restrict__ sigma_prime,
               const uint8_t *__restrict__ degenerate, const uint8_t *__restrict__ labels,
               double2 *__restrict__ rec, uint8_t *__restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double r44[G6R_REC_DOUBLES];
    for (int k = 0; k < 3; ++k) r44[k] = mu_p[3 * i + k];
    for (int k = 0; k < 3; ++k) r44[3 + k] = mu_d[3 * i + k];
    for (int k = 0; k < 9; ++k) r44[6 + k] = adjust[9 * i + k];
    const double *Q = prec + 9 * i;
    r44[15] = Q[0];
    r44[16] = Q[4];
    r44[17] = Q[8];
    r44[18] = Q[1];
    r44[19] = Q[2];
    r44[20] = Q[5];
    for (int k = 0; k < 9; ++k) r44[21 + k] = sigma_prime[9 * i + k];
    for (int k = 0; k < 12; ++k) r44[30 + k] = sh[12 * i + k];
    r44[42] = opacity[i];
    r44[43] = w_norm[i];
    put_record(rec, n, i, r44);
    flags[i] = (uint8_t)((labels[i] & 15u) | (degenerate[i] ? G6R_FLAG_DEGENERATE : 0u));
}

int launch_prepare(int64_t n, const double *mu_p, const double *mu_d, const double *cov_raw,
                   const double *sh, const double *opacity_raw, const uint8_t *labels,
                   const double *ss, double ds, int w_mode, double *records, uint8_t *flags,
                   int64_t *label_counts, cudaStream_t st) {
    if (cudaMemsetAsync(label_counts, 0, 32 * sizeof(int64_t), st) != cudaSuccess) return G6R_ECUDA;
    if (n == 0) return G6R_OK;
    // (2 pi)^-1.5 exactly as Python evaluates it (core.py:340)
    const double w_raw_const = pow(2.0 * 3.141592653589793, -1.5);
    k_prepare<<<(unsigned)ceil_div(n, kBlock), kBlock, 0, st>>>(
        n, mu_p, mu_d, cov_raw, sh, opacity_raw, labels, ss[0], ss[1], ss[2], ds, w_mode,
        w_raw_const, reinterpret_cast<double2 *>(records), flags,
        reinterpret_cast<unsigned long long *>(label_counts));
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_pack_records(int64_t n, const double *mu_p, const double *mu_d, const double *sh,
                        const double *opacity, const double *w_norm, const double *adjust,
                        const double *prec, const double *sigma_prime, const uint8_t *degenerate,
                        const uint8_t *labels, double *records, uint8_t *flags, cudaStream_t st) {
    if (n == 0) return G6R_OK;
    k_pack_records<<<(unsigned)ceil_div(n, kBlock), kBlock, 0, st>>>(
        n, mu_p, mu_d, sh, opacity, w_norm, adjust, prec, sigma_prime, degenerate, labels,
        reinterpret_cast<double2 *>(records), flags);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

// --- scene ingest: G6DS record block -> f64 SoA (sceneio.py:77-111) ---------
// One CTA stages 128 contiguous 168-byte records (21 KiB) through shared
// memory with coalesced 8-byte loads, then writes every output field with
// consecutive threads on consecutive output doubles.  HBM-bound: 168 B read
// and 320 B + 1 B written per Gaussian.
constexpr int kDecodeRecs = 128;
constexpr int kRecWords = 21;   // 168 bytes as u64

__global__ void __launch_bounds__(kBlock)
k_decode_records(int64_t n, const unsigned long long *__restrict__ recs, double *__restrict__ mu_p,
                 double *__restrict__ mu_d, double *__restrict__ cov_raw, double *__restrict__ sh,
                 double *__restrict__ opacity_raw, uint8_t *__restrict__ labels,
                 int32_t *__restrict__ bad) {
    __shared__ unsigned long long s[kDecodeRecs * kRecWords];
    const int64_t first = (int64_t)blockIdx.x * kDecodeRecs;
    const int cnt = (int)(n - first < kDecodeRecs ? n - first : kDecodeRecs);
    const unsigned long long *src = recs + first * kRecWords;
    for (int k = threadIdx.x; k < cnt * kRecWords; k += blockDim.x) s[k] = src[k];
    __syncthreads();
    const float *f = reinterpret_cast<const float *>(s);              // 42 floats per record
    const uint8_t *b = reinterpret_cast<const uint8_t *>(s);          // 168 bytes per record
    bool oops = false;
    struct Field { double *out; int off, width; };
    const Field fields[5] = {{mu_p, 0, 3}, {mu_d, 3, 3}, {cov_raw, 6, 21}, {sh, 27, 12},
                             {opacity_raw, 39, 1}};
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const Field fd = fields[q];
        for (int k = threadIdx.x; k < cnt * fd.width; k += blockDim.x) {
            const int r = k / fd.width, c = k - r * fd.width;
            const float v = f[r * 42 + fd.off + c];
            oops |= !isfinite(v);
            fd.out[first * fd.width + k] = (double)v;
        }
    }
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
        const uint8_t l = b[r * 168 + 160];
        oops |= l < 1 || l > 11;
        labels[first + r] = l;
    }
    if (__syncthreads_or(oops) && threadIdx.x == 0) *bad = 1;
}

int launch_decode_records(int64_t n, const void *recs, double *mu_p, double *mu_d, double *cov_raw,
                          double *sh, double *opacity_raw, uint8_t *labels, int32_t *bad,
                          cudaStream_t st) {
    if (n == 0) return 0;
    k_decode_records<<<(unsigned)ceil_div(n, kDecodeRecs), kBlock, 0, st>>>(
        n, static_cast<const unsigned long long *>(recs), mu_p, mu_d, cov_raw, sh, opacity_raw,
        labels, bad);
    return cudaGetLastError() != cudaSuccess;
}

}  // namespace g6r
