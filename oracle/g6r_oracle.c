/*
 * g6r_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference renderer's per-Gaussian and
 * per-pixel loops (splatct 0.1.0, /root/reference/pkg/src/splatct).  It is the
 * checker the CUDA path is compared against; nothing in the product package
 * links or calls it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.
 *
 * Built with -ffp-contract=off (no FMA contraction) so every expression rounds
 * exactly as the reference's Cython build does (setup.py:13).  Expression
 * association below follows the reference statement order; see the citations.
 *
 * Parity: pinned against the compiled reference (oracle/_ref) and the golden
 * fixtures in tests/golden (tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define STAGE_DRAWN 0
#define STAGE_VIEW_DEGENERATE 1
#define STAGE_DEPTH 3
#define STAGE_PROJECTION 4
#define STAGE_VIEWPORT 5

/* Slicing step of the 6D Gaussian against the unit view direction.
 * Reference: _kernels.pyx:190-229 (project_stage1), mirror _kernels_py.py:182-220.
 * Writes view, mean_adj, quad for rows whose camera distance is non-degenerate;
 * others get stage=1 and are left untouched. */
void or_project_stage1(int64_t n, const double *mu_p, const double *mu_d,
                       const double *adjust, const double *prec,
                       double px, double py, double pz,
                       double *view, double *mean_adj, double *quad,
                       uint8_t *stage)
{
    for (int64_t i = 0; i < n; ++i) {
        const double *p = mu_p + 3 * i;
        const double ex = p[0] - px, ey = p[1] - py, ez = p[2] - pz;
        const double len = sqrt(ex * ex + ey * ey + ez * ez);
        if (!(len > 1e-12)) {
            stage[i] = STAGE_VIEW_DEGENERATE;
            continue;
        }
        const double rl = 1.0 / len;
        const double v0 = ex * rl, v1 = ey * rl, v2 = ez * rl;
        const double *md = mu_d + 3 * i;
        const double g0 = v0 - md[0], g1 = v1 - md[1], g2 = v2 - md[2];
        const double *A = adjust + 9 * i;
        const double *Q = prec + 9 * i;
        view[3 * i + 0] = v0;
        view[3 * i + 1] = v1;
        view[3 * i + 2] = v2;
        /* row-wise (a0*g0 + a1*g1) + a2*g2, then added to mu_p (_kernels.pyx:215-223) */
        mean_adj[3 * i + 0] = p[0] + (A[0] * g0 + A[1] * g1 + A[2] * g2);
        mean_adj[3 * i + 1] = p[1] + (A[3] * g0 + A[4] * g1 + A[5] * g2);
        mean_adj[3 * i + 2] = p[2] + (A[6] * g0 + A[7] * g1 + A[8] * g2);
        /* Mahalanobis quadratic with the reference's association (:224-229) */
        const double diag = Q[0] * g0 * g0 + Q[4] * g1 * g1 + Q[8] * g2 * g2;
        const double off = Q[1] * g0 * g1 + Q[2] * g0 * g2 + Q[5] * g1 * g2;
        quad[i] = diag + 2.0 * off;
    }
}

static inline double clamp01(double c)
{
    if (c < 0.0) return 0.0;
    if (c > 1.0) return 1.0;
    return c;
}

/* Camera transform, degree-1 SH shading, EWA projection and screen culls for
 * rows still at stage 0.  Reference: _kernels.pyx:232-363, _kernels_py.py:223-325. */
void or_project_stage2(int64_t n, const double *view, const double *mean_adj,
                       const double *sh, const double *sigma_prime,
                       const double *rot, double px, double py, double pz,
                       double near_, double far_, double f, double ox, double oy,
                       double lim_x, double lim_y, double width, double height,
                       double low_pass, double sh_c0, double sh_c1,
                       double *means2d, double *conics, double *colors,
                       double *depths, int32_t *radii, uint8_t *stage)
{
    const double R00 = rot[0], R01 = rot[1], R02 = rot[2];
    const double R10 = rot[3], R11 = rot[4], R12 = rot[5];
    const double R20 = rot[6], R21 = rot[7], R22 = rot[8];
    for (int64_t i = 0; i < n; ++i) {
        if (stage[i] != STAGE_DRAWN) continue;
        const double *m = mean_adj + 3 * i;
        const double wx = m[0] - px, wy = m[1] - py, wz = m[2] - pz;
        const double cx = R00 * wx + R01 * wy + R02 * wz;
        const double cy = R10 * wx + R11 * wy + R12 * wz;
        const double cz = R20 * wx + R21 * wy + R22 * wz;
        if (!(cz >= near_ && cz <= far_)) {
            stage[i] = STAGE_DEPTH;
            continue;
        }
        /* degree-1 SH, basis-major [Y00, Y1-1, Y10, Y11] x RGB (:271-276) */
        const double *v = view + 3 * i;
        const double *c = sh + 12 * i;
        double rgb[3];
        for (int k = 0; k < 3; ++k)
            rgb[k] = clamp01(sh_c0 * c[k] - sh_c1 * v[1] * c[3 + k]
                             + sh_c1 * v[2] * c[6 + k] - sh_c1 * v[0] * c[9 + k] + 0.5);

        const double iz = 1.0 / cz;
        const double u = f * cx * iz + ox;
        const double w = f * cy * iz + oy;
        double xs = cx * iz;
        if (xs < -lim_x) xs = -lim_x;
        else if (xs > lim_x) xs = lim_x;
        xs = xs * cz;
        double ys = cy * iz;
        if (ys < -lim_y) ys = -lim_y;
        else if (ys > lim_y) ys = lim_y;
        ys = ys * cz;
        const double j00 = f * iz;
        const double j02 = -f * xs * iz * iz;
        const double j12 = -f * ys * iz * iz;

        /* B = S' R^T, then the six unique entries of R B (:309-323) */
        const double *S = sigma_prime + 9 * i;
        double B[3][3];
        for (int r = 0; r < 3; ++r) {
            B[r][0] = S[3 * r] * R00 + S[3 * r + 1] * R01 + S[3 * r + 2] * R02;
            B[r][1] = S[3 * r] * R10 + S[3 * r + 1] * R11 + S[3 * r + 2] * R12;
            B[r][2] = S[3 * r] * R20 + S[3 * r + 1] * R21 + S[3 * r + 2] * R22;
        }
        const double m00 = R00 * B[0][0] + R01 * B[1][0] + R02 * B[2][0];
        const double m01 = R00 * B[0][1] + R01 * B[1][1] + R02 * B[2][1];
        const double m02 = R00 * B[0][2] + R01 * B[1][2] + R02 * B[2][2];
        const double m11 = R10 * B[0][1] + R11 * B[1][1] + R12 * B[2][1];
        const double m12 = R10 * B[0][2] + R11 * B[1][2] + R12 * B[2][2];
        const double m22 = R20 * B[0][2] + R21 * B[1][2] + R22 * B[2][2];

        const double k00 = j00 * m00 + j02 * m02;
        const double k01 = j00 * m01 + j02 * m12;
        const double k02 = j00 * m02 + j02 * m22;
        const double k11 = j00 * m11 + j12 * m12;
        const double k12 = j00 * m12 + j12 * m22;
        const double ca = k00 * j00 + k02 * j02 + low_pass;
        const double cb = k01 * j00 + k02 * j12;
        const double cc = k11 * j00 + k12 * j12 + low_pass;
        const double det = ca * cc - cb * cb;
        if (!(isfinite(det) && det > 0.0 && isfinite(u) && isfinite(w))) {
            stage[i] = STAGE_PROJECTION;
            continue;
        }
        const double idet = 1.0 / det;
        double rx = ceil(3.0 * sqrt(ca));
        if (rx > 1048576.0) rx = 1048576.0;
        double ry = ceil(3.0 * sqrt(cc));
        if (ry > 1048576.0) ry = 1048576.0;
        /* x86 cvttsd2si yields INT32_MIN for NaN; keep that explicit */
        const int32_t irx = isnan(rx) ? INT32_MIN : (int32_t)rx;
        const int32_t iry = isnan(ry) ? INT32_MIN : (int32_t)ry;
        if (!(u + irx >= 0.0 && u - irx <= width - 1.0
              && w + iry >= 0.0 && w - iry <= height - 1.0)) {
            stage[i] = STAGE_VIEWPORT;
            continue;
        }
        means2d[2 * i] = u;
        means2d[2 * i + 1] = w;
        conics[3 * i] = cc * idet;
        conics[3 * i + 1] = -cb * idet;
        conics[3 * i + 2] = ca * idet;
        colors[3 * i] = rgb[0];
        colors[3 * i + 1] = rgb[1];
        colors[3 * i + 2] = rgb[2];
        depths[i] = cz;
        radii[2 * i] = irx;
        radii[2 * i + 1] = iry;
    }
}

/* Front-to-back over-compositing of depth-sorted tile runs.
 * Reference: _kernels.pyx:36-105 (fused f32/f64), _kernels_py.py:45-103.
 * Pixels of empty tiles keep the caller-initialised background. */
#define DEFINE_COMPOSITE(NAME, REAL, EXPF)                                          \
void NAME(const REAL *means2d, const REAL *conics, const REAL *colors,              \
          const REAL *alphas, const int32_t *entry_splat,                           \
          const int64_t *tile_starts, int64_t n_tiles, int tiles_x, int tile_size,  \
          int width, int height, REAL *image, REAL *final_t, int32_t *last_contrib) \
{                                                                                   \
    const REAL skip_lo = (REAL)-4.5, floor_a = (REAL)(1.0 / 255.0);                 \
    const REAL t_stop = (REAL)1e-4, half = (REAL)-0.5;                              \
    for (int64_t t = 0; t < n_tiles; ++t) {                                         \
        const int64_t lo = tile_starts[t], hi = tile_starts[t + 1];                 \
        if (lo == hi) continue;                                                     \
        const int x0 = (int)(t % tiles_x) * tile_size;                              \
        const int y0 = (int)(t / tiles_x) * tile_size;                              \
        const int x1 = x0 + tile_size < width ? x0 + tile_size : width;             \
        const int y1 = y0 + tile_size < height ? y0 + tile_size : height;           \
        for (int y = y0; y < y1; ++y) {                                             \
            for (int x = x0; x < x1; ++x) {                                         \
                const REAL fx = (REAL)x, fy = (REAL)y;                              \
                REAL T = 1, r = 0, g = 0, b = 0, a = 0;                             \
                int last = 0;                                                       \
                for (int64_t e = lo; e < hi; ++e) {                                 \
                    const int64_t s = entry_splat[e];                               \
                    const REAL dx = fx - means2d[2 * s];                            \
                    const REAL dy = fy - means2d[2 * s + 1];                        \
                    const REAL *q = conics + 3 * s;                                 \
                    const REAL pw = half * (q[0] * dx * dx + q[2] * dy * dy)        \
                                    - q[1] * dx * dy;                               \
                    if (pw > 0 || pw < skip_lo) continue;                           \
                    const REAL ai = alphas[s] * EXPF(pw);                           \
                    if (ai < floor_a) continue;                                     \
                    const REAL wgt = ai * T;                                        \
                    r = r + colors[3 * s] * wgt;                                    \
                    g = g + colors[3 * s + 1] * wgt;                                \
                    b = b + colors[3 * s + 2] * wgt;                                \
                    a = a + wgt;                                                    \
                    T = T * (1 - ai);                                               \
                    last = (int)(e - lo) + 1;                                       \
                    if (T < t_stop) break;                                          \
                }                                                                   \
                const int64_t p = (int64_t)y * width + x;                           \
                image[4 * p] = r;                                                   \
                image[4 * p + 1] = g;                                               \
                image[4 * p + 2] = b;                                               \
                image[4 * p + 3] = a;                                               \
                final_t[p] = T;                                                     \
                last_contrib[p] = last;                                             \
            }                                                                       \
        }                                                                           \
    }                                                                               \
}

/* glibc 2.39 expf restated (third-party dependency of the reference's f32
 * compositor, _kernels.pyx:29-33 -> libm expf; sysdeps/ieee754/flt-32/e_expf.c
 * with the x86-64 FMA variant's contractions).  The table is 2^(i/32) rounded
 * to double minus (i << 47).  tests/test_oracle.py pins this model against the
 * host libm; the CUDA compositor implements the same arithmetic. */
static uint64_t expf_tab[32];
static int expf_tab_ready = 0;
float or_expf_glibc(float x)
{
    if (!expf_tab_ready) {
        for (int i = 0; i < 32; ++i) {
            double v = exp2((double)i / 32.0);
            uint64_t u;
            memcpy(&u, &v, 8);
            expf_tab[i] = u - ((uint64_t)i << 47);
        }
        expf_tab_ready = 1;
    }
    const double inv_ln2_n = 0x1.71547652b82fep+5, shift = 0x1.8p+52;
    const double c0 = 0x1.c6af84b912394p-20, c1 = 0x1.ebfce50fac4f3p-13, c2 = 0x1.62e42ff0c52d6p-6;
    const double xd = (double)x;
    const double z = inv_ln2_n * xd;
    double kd = z + shift;
    uint64_t ki;
    memcpy(&ki, &kd, 8);
    kd -= shift;
    const double r = fma(inv_ln2_n, xd, -kd);
    uint64_t t = expf_tab[ki % 32] + (ki << 47);
    double s;
    memcpy(&s, &t, 8);
    const double p = fma(c0, r, c1);
    const double r2 = r * r;
    double y = fma(c2, r, 1.0);
    y = fma(p, r2, y);
    y = y * s;
    return (float)y;
}

/* The host libm exp over an array (checker for the device's restated glibc
 * exp used by the f64 compositors; the reference's f64 kernel and its
 * brute-force oracle call this same libm exp). */
void or_libm_exp_batch(int64_t n, const double *x, double *y)
{
    for (int64_t i = 0; i < n; ++i) y[i] = exp(x[i]);
}

void or_expf_glibc_batch(int64_t n, const float *x, float *y)
{
    for (int64_t i = 0; i < n; ++i) y[i] = or_expf_glibc(x[i]);
}

/* out[i] = fma(a[i], b[i], c[i]), correctly rounded (C99 fma).  The reference's
 * (N,3) @ (3,3) world-coordinate matmul (priming.py:134) runs through OpenBLAS
 * dgemm, which on the reference host accumulates fma(q2,d2, fma(q1,d1, q0*d0)). */
void or_fma_batch(int64_t n, const double *a, const double *b, const double *c, double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = fma(a[i], b[i], c[i]);
}

DEFINE_COMPOSITE(or_composite_f32, float, expf)
DEFINE_COMPOSITE(or_composite_f64, double, exp)

/* Adjoint of the f64 compositor: per-entry gradient rows (E, 9) in the order
 * mean_x, mean_y, conic_a, conic_b, conic_c, r, g, b, alpha.
 * Reference: _kernels.pyx:108-187, _kernels_py.py:106-179. */
void or_composite_backward(const double *means2d, const double *conics,
                           const double *colors, const double *alphas,
                           const int32_t *entry_splat, const int64_t *tile_starts,
                           int64_t n_tiles, int tiles_x, int tile_size, int width,
                           int height, const double *final_t,
                           const int32_t *last_contrib, const double *grad_image,
                           double *entry_grads)
{
    for (int64_t t = 0; t < n_tiles; ++t) {
        const int64_t lo = tile_starts[t];
        const int x0 = (int)(t % tiles_x) * tile_size;
        const int y0 = (int)(t / tiles_x) * tile_size;
        const int x1 = x0 + tile_size < width ? x0 + tile_size : width;
        const int y1 = y0 + tile_size < height ? y0 + tile_size : height;
        for (int y = y0; y < y1; ++y) {
            for (int x = x0; x < x1; ++x) {
                const int64_t p = (int64_t)y * width + x;
                const int last = last_contrib[p];
                if (last == 0) continue;
                const double gr = grad_image[4 * p], gg = grad_image[4 * p + 1];
                const double gb = grad_image[4 * p + 2], ga = grad_image[4 * p + 3];
                if (gr == 0.0 && gg == 0.0 && gb == 0.0 && ga == 0.0) continue;
                const double fx = (double)x, fy = (double)y;
                double T = final_t[p];
                double sr = 0.0, sg = 0.0, sb = 0.0, sa = 0.0;
                for (int64_t e = lo + last - 1; e >= lo; --e) {
                    const int64_t s = entry_splat[e];
                    const double dx = fx - means2d[2 * s];
                    const double dy = fy - means2d[2 * s + 1];
                    const double qa = conics[3 * s], qb = conics[3 * s + 1], qc = conics[3 * s + 2];
                    const double pw = -0.5 * (qa * dx * dx + qc * dy * dy) - qb * dx * dy;
                    if (pw > 0.0 || pw < -4.5) continue;
                    const double ge = exp(pw);
                    const double ai = alphas[s] * ge;
                    if (ai < 1.0 / 255.0) continue;
                    const double om = 1.0 - ai;
                    T = T / om;
                    const double wgt = ai * T;
                    double *eg = entry_grads + 9 * e;
                    const double *col = colors + 3 * s;
                    eg[5] += wgt * gr;
                    eg[6] += wgt * gg;
                    eg[7] += wgt * gb;
                    const double dai = T * (col[0] * gr + col[1] * gg + col[2] * gb + ga)
                                       - (sr * gr + sg * gg + sb * gb + sa * ga) / om;
                    eg[8] += ge * dai;
                    const double dp = ai * dai;
                    eg[0] += dp * (qa * dx + qb * dy);
                    eg[1] += dp * (qc * dy + qb * dx);
                    eg[2] += dp * (-0.5 * dx * dx);
                    eg[3] += dp * (-dx * dy);
                    eg[4] += dp * (-0.5 * dy * dy);
                    sr = sr + col[0] * wgt;
                    sg = sg + col[1] * wgt;
                    sb = sb + col[2] * wgt;
                    sa = sa + wgt;
                }
            }
        }
    }
}
