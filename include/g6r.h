/*
 * g6r.h -- C ABI of the B200-native 6DGS render path (libg6r.so).
 *
 * Drop-in for the render hot path of the reference package splatct 0.1.0
 * (arXiv 2505.17338 "Render-FM"): per-view 6D->3D slicing, EWA projection and
 * SH shading, tile binning, sort, range extraction and front-to-back alpha
 * compositing.  Every pointer argument is a DEVICE pointer unless marked
 * "host"; every call is asynchronous on the given stream and only enqueues
 * work (no device synchronisation, no allocation).  Calls are re-entrant:
 * concurrent callers need distinct workspaces (or distinct streams ordered by
 * the caller).  No torch types cross this boundary.
 *
 * Return codes: G6R_OK, or a negative code; g6r_last_error() (thread-local)
 * then describes the failure.  Mapping used by the Python host
 * (paper_2505_17338_b200/raster.py):
 *   G6R_EINVAL -> InvalidParameterError, G6R_ENOSPC -> retry with more entry
 *   capacity, G6R_ECUDA -> RuntimeError.
 *
 * Reference interfaces replaced (file:line in /root/reference/pkg/src/splatct):
 *   g6r_prepare          raster.py:120-137 prepare_scene (core.py:255-351)
 *   g6r_project          raster.py:229-309 _project_rows / project_scene,
 *                        _kernels.pyx:190-363 project_stage1/2 fused with the
 *                        opacity modulation (raster.py:258-261) and compaction
 *   g6r_project_stage1   _kernels.pyx:190-229 (kernel-module contract)
 *   g6r_project_stage2   _kernels.pyx:232-363 (kernel-module contract)
 *   g6r_bin              raster.py:340-381 bin_splats
 *   g6r_composite        raster.py:392-415 _composite / _kernels.pyx:36-105
 *   g6r_composite_backward _kernels.pyx:108-187
 *   g6r_render           raster.py:443-466 render_with_state / render
 *   g6r_render_views     many views of one scene (batched, pipelined)
 *   g6r_render_backward  diffrender.py:401-439 render_backward + :183-398 _backward_rows
 *     (= g6r_backward_forward + g6r_backward_apply)
 *   g6r_loss_grad        diffrender.py:117-138 _loss_parts, _ssim.py:123-201
 *   g6r_adam_step        diffrender.py:481-509 adam_step
 *   g6r_decode_records   sceneio.py:77-111 load_scene (record block)
 *   g6r_decode_param_volume  priming.py:232-285 decode_param_volume
 *   g6r_filter_rows      priming.py:362-374 filter_scene
 *   g6r_frame.rgba8      metrics.py:21-25 composite_over + _png.py:21-32 to_rgba_u8
 */
#ifndef G6R_H_
#define G6R_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *g6r_stream_t; /* == cudaStream_t */

#define G6R_OK 0
#define G6R_EINVAL (-22)
#define G6R_ENOSPC (-28)
#define G6R_ECUDA (-5)

/* Per-Gaussian prepared record: 44 doubles stored as 22 columns of
 * 16-byte (double2) packets, column-major over Gaussians: element (c, i) of
 * the record block is the double2 at records[2*(c*n + i)].  Packet order:
 *   mu_p[0..2], mu_d[0..2], adjust[9] (row-major), precision_dd
 *   (00,11,22,01,02,12), sigma_prime[9] (row-major), sh[12], opacity, w_norm. */
#define G6R_REC_DOUBLES 44
#define G6R_REC_COLUMNS 22

/* flags byte per Gaussian: bits 0..3 group label, bit 7 degenerate. */
#define G6R_FLAG_DEGENERATE 0x80u

/* counters written by g6r_project / g6r_render / g6r_bin (int64 device array
 * of G6R_NCOUNTERS): */
enum {
    G6R_CNT_DRAWN = 0,        /* M: splats kept */
    G6R_CNT_ENTRIES = 1,      /* E: tile entries (also when over capacity) */
    G6R_CNT_FATE = 2,         /* [2..7]: stage-code histogram 0..5 of selected rows */
    G6R_CNT_OVERFLOW = 8,     /* 1 if E exceeded entry_capacity (nothing sorted) */
    G6R_CNT_GRAD_NONFINITE = 9, /* g6r_backward_apply / g6r_render_backward: 1 if any
                                   gradient element written is not finite, else 0 */
    G6R_NCOUNTERS = 16
};

typedef struct g6r_camera {
    double position[3];
    double rotation[9];  /* row-major world->camera (camera.py:18-62) */
    double focal;        /* pixels, fx == fy */
    double cx, cy;       /* principal point, pixels */
    double znear, zfar;
    int32_t width, height;
} g6r_camera;

typedef struct g6r_config {
    int32_t tile_size;   /* 1..32 (raster.py:89) */
    int32_t precision;   /* 0: f32 framebuffer, 1: f64 (raster.py:93) */
    double low_pass;     /* px^2 added to the cov2d diagonal (raster.py:90) */
    double alpha_max;    /* per-splat alpha cap (raster.py:91) */
    /* Compositor exp in the f32 framebuffer: 0 = glibc expf restated exactly
     * (framebuffer bit-identical to the reference's, _kernels.pyx:29-33);
     * 1 = SFU ex2 (image within ~1e-6 relative of mode 0, far inside the
     * 1e-3 max-abs / 60 dB PSNR parity bound; every alpha-floor decision is
     * still exact).  Ignored for f64 and for RGBA8 frames (always exact). */
    int32_t exp_mode;
    int32_t reserved;    /* 0 */
} g6r_config;

/* Device-resident scene after g6r_prepare. */
typedef struct g6r_scene {
    int64_t n;
    const double *records;  /* G6R_REC_DOUBLES * n doubles, layout above */
    const uint8_t *flags;   /* n */
} g6r_scene;

/* Optional SplatBatch-shaped outputs of the projection (raster.py:157-170),
 * compacted in ascending scene order; each pointer may be NULL.  Capacity n. */
typedef struct g6r_splat_out {
    int64_t *gids;      /* (M)   scene row */
    double *means2d;    /* (M,2) */
    double *conics;     /* (M,3) */
    double *colors;     /* (M,3) */
    double *alphas;     /* (M)   */
    double *depths;     /* (M)   */
    int32_t *radii;     /* (M,2) */
    uint8_t *stage;     /* (n)   per scene row: 0 drawn, 1..5 cull, 255 unselected */
} g6r_splat_out;

/* Frame outputs of g6r_render. image is (H,W,4) premultiplied RGBA and
 * final_t (H,W), both float or double per config.precision; last_contrib is
 * (H,W) int32.  entry_splat (E) / tile_starts (T+1) are optional copies of the
 * sorted tile runs (raster.py:201-208). */
typedef struct g6r_frame {
    void *image;            /* required unless rgba8 is given */
    void *final_t;
    int32_t *last_contrib;
    int64_t *counters;      /* G6R_NCOUNTERS, required */
    int32_t *entry_splat;   /* optional, capacity entry_capacity */
    int64_t *tile_starts;   /* optional, T+1 */
    /* optional served-frame output fused into the compositor epilogue:
     * (H,W,4) u8 = round(clip(rgb + background * (1 - alpha), 0, 1) * 255),
     * alpha 255 (metrics.py:21-25 composite_over, _png.py:21-32 to_rgba_u8). */
    uint8_t *rgba8;
    double background[3];
    /* Optional page-locked host copies of image / rgba8.  g6r_render_views
     * copies each view on an internal copy stream as soon as the compositor
     * has finished that view (a device flag gates the copy), so the transfer
     * overlaps the rest of the call's rendering; the call stays ordered on its
     * stream (the copies are joined back before it returns). */
    void *host_image;
    uint8_t *host_rgba8;
} g6r_frame;

const char *g6r_version(void);
const char *g6r_last_error(void);

/* Prepared-scene storage: bytes for records of n Gaussians. */
size_t g6r_records_bytes(int64_t n);

/* View-independent slicing terms from raw parameters (raster.py:120-137).
 * mu_p, mu_d (n,3), cov_raw (n,21), sh (n,12), opacity_raw (n) f64; labels (n) u8.
 * w_mode 0 = "peak", 1 = "raw".  label_counts (device int64[32]) receives
 * per-label totals [0..15] and per-label degenerate counts [16..31] so the
 * host can apply the degenerate policy (raster.py:431-440) with no per-frame
 * transfer. */
int g6r_prepare(int64_t n, const double *mu_p, const double *mu_d,
                const double *cov_raw, const double *sh, const double *opacity_raw,
                const uint8_t *labels, const double *spatial_scale /* host (3) */,
                double directional_scale, int32_t w_mode,
                double *records, uint8_t *flags, int64_t *label_counts,
                g6r_stream_t stream);

/* Pack externally computed terms (e.g. the CPU oracle's) into the record
 * layout, for isolated projection checks.  adjust, precision_dd, sigma_prime
 * are (n,3,3) row-major. */
int g6r_pack_records(int64_t n, const double *mu_p, const double *mu_d,
                     const double *sh, const double *opacity, const double *w_norm,
                     const double *adjust, const double *precision_dd,
                     const double *sigma_prime, const uint8_t *degenerate,
                     const uint8_t *labels, double *records, uint8_t *flags,
                     g6r_stream_t stream);

/* Workspace bytes for one in-flight view of an n-Gaussian scene with
 * `tiles` tiles and room for `entry_capacity` tile entries. */
size_t g6r_workspace_bytes(int64_t n, int64_t tiles, int64_t entry_capacity,
                           int32_t precision);

/* Full forward render of one view (raster.py:443-466).  group_mask: bit g set
 * = render group g (bit 0..11); 0xFFF = everything (group_mask=None).
 * On G6R_ENOSPC-style overflow the counters report E and OVERFLOW=1; the
 * call still returns G6R_OK (the condition is only known on the device) and
 * the frame must be re-rendered with entry_capacity >= E. */
int g6r_render(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
               const g6r_config *cfg, void *workspace, size_t workspace_bytes,
               int64_t entry_capacity, const g6r_frame *frame,
               const g6r_splat_out *splats /* may be NULL */, g6r_stream_t stream);

/* Stage timing: a profiler records CUDA events around each stage of every
 * view rendered through g6r_render_views (on the render stream, so the
 * timed region is the real one).  Stages: 0 project (slice+project+compact+
 * duplicate), 1 sort (histogram + radix passes), 2 ranges, 3 composite. */
#define G6R_NSTAGES 4
typedef struct g6r_profiler g6r_profiler;
g6r_profiler *g6r_profiler_create(int32_t max_views);
void g6r_profiler_destroy(g6r_profiler *prof);
void g6r_profiler_reset(g6r_profiler *prof);
/* Synchronises on the recorded events; stage_ms[G6R_NSTAGES] receives the
 * summed per-stage milliseconds, *views the number of views recorded. */
int g6r_profiler_read(g6r_profiler *prof, double *stage_ms, int32_t *views);

/* Render `count` views of one scene (same image size) into frames[k], in
 * batches of `batch` views (1..16): every stage kernel processes a whole batch
 * per launch (grid = work x views), so one view's long tile runs overlap the
 * other views' work and the projection shares the record stream through L2.
 * The workspace must hold batch x g6r_workspace_bytes(...).  When it holds
 * twice that, there is more than one batch and prof is NULL, consecutive
 * batches alternate between the two halves on two internal streams forked from
 * and joined back into `stream` (a batch's projection and sort overlap the
 * previous batch's compositing); the call stays asynchronous and ordered on
 * `stream`.  final_t / last_contrib may be NULL in these frames.  prof may be
 * NULL; it records one slot per batch (and keeps the batches on one stream). */
int g6r_render_views(const g6r_scene *scene, uint32_t group_mask,
                     const g6r_camera *cams /* host array */, int32_t count,
                     const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                     int64_t entry_capacity, const g6r_frame *frames /* host array */,
                     int32_t batch, g6r_profiler *prof, g6r_stream_t stream);

/* Backward render (diffrender.py:401-439 render_backward): an f64 forward of
 * the view followed by the adjoint compositor, the per-splat reduction and the
 * chain to the raw parameters (diffrender.py:183-398).  grad_image is
 * d loss / d image (H,W,4) f64; the gradient arrays (scene rows, shapes as the
 * raw scene: (n,3) (n,3) (n,21) (n,12) (n)) are fully overwritten -- culled,
 * masked and degenerate Gaussians get exact zeros.  cfg->precision must be 1
 * and cfg->tile_size 16.  mu_p/mu_d/cov_raw/sh are the scene's raw device
 * arrays (the factor L is rebuilt from cov_raw); spatial_scale is host (3).
 * image_out (optional, (H,W,4) f64) receives the forward image.  Deterministic:
 * no floating-point atomics. */
size_t g6r_backward_workspace_bytes(int64_t n, int32_t width, int32_t height, int32_t tile_size,
                                    int64_t entry_capacity);
int g6r_render_backward(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
                        const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                        int64_t entry_capacity, const double *mu_p, const double *mu_d,
                        const double *cov_raw, const double *sh,
                        const double *spatial_scale /* host (3) */, double directional_scale,
                        int32_t w_mode, const double *grad_image, double *g_mu_p, double *g_mu_d,
                        double *g_cov_raw, double *g_sh, double *g_opacity_raw, int64_t *counters,
                        double *image_out, g6r_stream_t stream);

/* The two halves of g6r_render_backward, for loops that compute the loss
 * between them (the fine-tune loop): the f64 forward keeps its state
 * (sorted runs, final_t, last_contrib, splat rows) in the workspace and writes
 * the image to image_out; apply then runs the adjoint on that state.  Both
 * calls must see the same scene, camera, config and entry_capacity. */
int g6r_backward_forward(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
                         const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                         int64_t entry_capacity, int64_t *counters, double *image_out,
                         g6r_stream_t stream);
int g6r_backward_apply(const g6r_scene *scene, const g6r_camera *cam, const g6r_config *cfg,
                       void *workspace, size_t workspace_bytes, int64_t entry_capacity,
                       const double *mu_p, const double *mu_d, const double *cov_raw,
                       const double *sh, const double *spatial_scale /* host (3) */,
                       double directional_scale, int32_t w_mode, const double *grad_image,
                       double *g_mu_p, double *g_mu_d, double *g_cov_raw, double *g_sh,
                       double *g_opacity_raw, int64_t *counters, g6r_stream_t stream);

/* Scene ingest (sceneio.py:77-111): decode `n` G6DS 168-byte records (the
 * block after the 168-byte file header, already in device memory, 8-byte
 * aligned) into the f64 SoA scene arrays (n,3) (n,3) (n,21) (n,12) (n) and
 * labels (n).  Sets *bad (device int32) to 1 if any parameter is not finite or
 * a label lies outside [1, 11]. */
int g6r_decode_records(int64_t n, const void *records, double *mu_p, double *mu_d,
                       double *cov_raw, double *sh, double *opacity_raw, uint8_t *labels,
                       int32_t *bad, g6r_stream_t stream);

/* Order-preserving stream compaction scratch for n items (Psi decode over
 * the half-grid voxels, group filter over scene rows). */
size_t g6r_compact_workspace_bytes(int64_t n);

/* Psi decode (priming.py:232-285 decode_param_volume) in two calls: count the
 * foreground voxels of the half grid (dims = D', H', W'; labels_half (V) u8 =
 * labels[::2, ::2, ::2][:D', :H', :W']), writing *count (device int64) and the
 * per-chunk offsets into the workspace; the caller sizes the outputs, then
 * decode emits the scene rows in np.nonzero order.  psi is (37, V) f32
 * (psi_f32=1, the .raw file precision) or f64; base_rgba (4, V) f64 are input
 * channels 2..5 on the half grid; spacing, origin (3) and direction (3x3,
 * row-major) are host arrays.  Outputs as the scene SoA: (count,3) (count,3)
 * (count,21) (count,12) (count) and labels (count). */
int g6r_decode_param_volume_count(const int32_t *dims /* host (3) */, const uint8_t *labels_half,
                                  void *workspace, size_t workspace_bytes, int64_t *count,
                                  g6r_stream_t stream);
int g6r_decode_param_volume(const int32_t *dims /* host (3) */, const void *psi, int32_t psi_f32,
                            const double *base_rgba, const uint8_t *labels_half,
                            const double *spacing, const double *origin, const double *direction,
                            void *workspace, size_t workspace_bytes, double *mu_p, double *mu_d,
                            double *cov_raw, double *sh, double *opacity_raw, uint8_t *labels,
                            g6r_stream_t stream);

/* Group filter (priming.py:362-374 filter_scene): rows whose label bit is set
 * in group_mask, in scene order, into outputs of capacity n; *count (device
 * int64) receives the kept row count. */
int g6r_filter_rows(int64_t n, const uint8_t *labels, uint32_t group_mask, const double *mu_p,
                    const double *mu_d, const double *cov_raw, const double *sh,
                    const double *opacity_raw, void *workspace, size_t workspace_bytes,
                    double *out_mu_p, double *out_mu_d, double *out_cov_raw, double *out_sh,
                    double *out_opacity_raw, uint8_t *out_labels, int64_t *count,
                    g6r_stream_t stream);

/* Photometric loss lambda_l1 * L1 + lambda_ssim * (1 - MS-SSIM) on the RGB
 * channels and its gradient with respect to the rendered image
 * (diffrender.py:117-138 _loss_parts, _ssim.py:123-201 ms_ssim_with_grad).
 * pred is (H,W,4) f64 on the device, target (H,W,target_channels) f64 with
 * target_channels 3 or 4; grad_out (H,W,4) is fully written (alpha slot 0).
 * weights (host, `scales` entries) are normalised here over the effective
 * scale count; images under 2^(scales-1)*11 px per side use single-scale
 * SSIM.  parts (host, 3) = {total, l1, ssim_loss}.  Synchronises the stream
 * (the scalar reductions are read back).  Deterministic.  The kernel sequence
 * is captured into a CUDA graph on first use for a given (workspace, size,
 * weights) and replayed afterwards; pred/target/grad_out are staged through
 * the workspace, so any caller buffers work. */
size_t g6r_loss_workspace_bytes(int32_t width, int32_t height);
int g6r_loss_grad(const double *pred, const double *target, int32_t target_channels,
                  int32_t width, int32_t height, double lambda_l1, double lambda_ssim,
                  int32_t scales, const double *weights, void *workspace, size_t workspace_bytes,
                  double *grad_out, double *parts, g6r_stream_t stream);

/* One bias-corrected Adam update of `count` f64 parameters in place
 * (diffrender.py:481-509, betas 0.9/0.999, eps 1e-8, the reference's operation
 * order): m, v are the moment buffers; lr is this group's learning rate;
 * bias1 = 1 - 0.9^t, bias2 = 1 - 0.999^t. */
int g6r_adam_step(int64_t count, double *param, const double *grad, double *m, double *v,
                  double lr, double bias1, double bias2, g6r_stream_t stream);

/* Sets *flag (device int32) to 1 if any of `count` doubles is not finite;
 * leaves it unchanged otherwise (GradientBuffer.all_finite, diffrender.py:179). */
int g6r_any_nonfinite(int64_t count, const double *x, int32_t *flag, g6r_stream_t stream);

/* Launch trace: with G6R_TRACE=1 in the environment every kernel launch is
 * followed by a CUDA event; this writes "label,ms" rows (device time between
 * consecutive launches' completions) to `path` (stderr if NULL) and clears the
 * trace.  Synchronises on the last event. */
int g6r_trace_dump(const char *path);

/* Zero-copy outputs: the device address of page-locked host memory (the
 * same pointer on unified-addressing systems).  A g6r_frame's image / rgba8
 * may point into such memory: the compositor epilogue then writes each
 * finished pixel over PCIe while the rest of the batch still renders, so host
 * images need no separate device->host copy after the render.  G6R_EINVAL if
 * `host` is not page-locked memory visible to the current device. */
int g6r_host_device_pointer(void *host, void **device);

/* Test probe: y[i] = the device expf used by the f32 compositor (glibc
 * algorithm, g6r_common.cuh) for n floats. */
int g6r_debug_expf(int64_t n, const float *x, float *y, g6r_stream_t stream);

/* Test probe: y[i] = the device exp used by the f64 compositors (glibc 2.39's
 * FMA exp restated, g6r_common.cuh exp_glibc) for n doubles in (-512, 512). */
int g6r_debug_exp(int64_t n, const double *x, double *y, g6r_stream_t stream);

/* Stage entry points with external inputs (the reference stage helpers). */
int g6r_project(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
                const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                int64_t *counters, const g6r_splat_out *splats, g6r_stream_t stream);

int g6r_bin(int64_t m, const double *means2d, const int32_t *radii, const double *depths,
            int32_t width, int32_t height, int32_t tile_size, void *workspace,
            size_t workspace_bytes, int64_t entry_capacity, int32_t *entry_splat,
            int64_t *tile_starts, int64_t *counters, g6r_stream_t stream);

/* precision 0: float inputs/outputs, 1: double. */
int g6r_composite(int64_t m, int32_t precision, const void *means2d, const void *conics,
                  const void *colors, const void *alphas, const int32_t *entry_splat,
                  const int64_t *tile_starts, int32_t tiles_x, int32_t tiles_y,
                  int32_t tile_size, int32_t width, int32_t height, void *workspace,
                  size_t workspace_bytes, void *image, void *final_t,
                  int32_t *last_contrib, g6r_stream_t stream);

/* Kernel-module contract mirrors (_kernels.pyx:190-363), f64 arrays. */
int g6r_project_stage1(int64_t n, const double *mu_p, const double *mu_d,
                       const double *adjust, const double *precision_dd,
                       double px, double py, double pz, double *view,
                       double *mean_adj, double *quad, uint8_t *stage,
                       g6r_stream_t stream);

int g6r_project_stage2(int64_t n, const double *view, const double *mean_adj,
                       const double *sh, const double *sigma_prime,
                       const double *rot /* host (9) */, double px, double py, double pz,
                       double znear, double zfar, double f, double ox, double oy,
                       double lim_x, double lim_y, double width, double height,
                       double low_pass, double sh_c0, double sh_c1, double *means2d,
                       double *conics, double *colors, double *depths, int32_t *radii,
                       uint8_t *stage, g6r_stream_t stream);

/* Adjoint of the f64 compositor (_kernels.pyx:108-187): per-entry gradient
 * rows entry_grads (E,9) = d/d(mean_x, mean_y, conic_a, conic_b, conic_c, r,
 * g, b, alpha), accumulated (+=) like the reference. */
int g6r_composite_backward(int64_t m, const double *means2d, const double *conics,
                           const double *colors, const double *alphas,
                           const int32_t *entry_splat, const int64_t *tile_starts,
                           int32_t tiles_x, int32_t tiles_y, int32_t tile_size,
                           int32_t width, int32_t height, const double *final_t,
                           const int32_t *last_contrib, const double *grad_image,
                           double *entry_grads, g6r_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* G6R_H_ */
