// g6r_internal.h -- host-side launchers shared between the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/g6r.h"

namespace g6r {

// Workspace carve-up for one view (see g6r_api.cu::layout).
struct Workspace {
    long long *internal;            // kNumInternal int64 (tickets)
    unsigned long long *proj_agg_m, *proj_agg_e, *proj_inc_m, *proj_inc_e;  // lookback, per projection block
    void *payload;                  // n compositing payloads (f32 or f64)
    unsigned long long *keys[2];    // entry keys, ping-pong
    unsigned *vals[2];              // entry values (splat index), ping-pong
    unsigned *hist;                 // kMaxPasses x kBins digit counts
    unsigned *sort_status;          // kMaxPasses x tiles_cap x kBins lookback words
    int64_t *tile_starts;           // T+1 (internal copy)
    int64_t entry_capacity;
    int64_t sort_tiles_cap;
};

struct ViewParams {
    double pos[3];
    double rot[9];
    double focal, cx, cy, znear, zfar, lim_x, lim_y, width, height;
    double low_pass, alpha_max;
    int32_t iw, ih, tile_size, tiles_x, tiles_y, precision;
};

int launch_prepare(int64_t n, const double *mu_p, const double *mu_d, const double *cov_raw,
                   const double *sh, const double *opacity_raw, const uint8_t *labels,
                   const double *ss, double ds, int w_mode, double *records, uint8_t *flags,
                   int64_t *label_counts, cudaStream_t st);
int launch_pack_records(int64_t n, const double *mu_p, const double *mu_d, const double *sh,
                        const double *opacity, const double *w_norm, const double *adjust,
                        const double *prec, const double *sigma_prime, const uint8_t *degenerate,
                        const uint8_t *labels, double *records, uint8_t *flags, cudaStream_t st);

// fused slice+project+compact+duplicate; writes counters[M,E,fate,overflow]
int launch_project(const g6r_scene &scene, uint32_t mask, const ViewParams &vp,
                   const Workspace &ws, int64_t *counters, const g6r_splat_out *splats,
                   bool write_entries, cudaStream_t st);
// binning of external splats (count, scan, duplicate) into ws.keys[0]/vals[0]
int launch_duplicate(int64_t m, const double *means2d, const int32_t *radii, const double *depths,
                     const ViewParams &vp, const Workspace &ws, int64_t *counters, cudaStream_t st);
// radix sort of ws.keys[0]/vals[0] (E read from counters); *final_buf receives
// the index (0/1) of the buffer holding the sorted result.
int launch_sort(const ViewParams &vp, const Workspace &ws, const int64_t *counters, cudaStream_t st);
// per-tile ranges into ws.tile_starts (+ optional copies of starts / entry_splat)
int launch_ranges(const ViewParams &vp, const Workspace &ws, const int64_t *counters,
                  int64_t *tile_starts_out, int32_t *entry_splat_out, cudaStream_t st);
int launch_debug_expf(int64_t n, const float *x, float *y, cudaStream_t st);
int launch_pack_payload(int64_t m, int precision, const void *means2d, const void *conics,
                        const void *colors, const void *alphas, void *payload, cudaStream_t st);
// entry values: vals0, or (sel != NULL) the sorted ping-pong buffer sel picks
int launch_composite(const ViewParams &vp, const void *payload, const unsigned *vals0,
                     const unsigned *vals1, const long long *sel, const int64_t *tile_starts, void *image, void *final_t,
                     int32_t *last_contrib, cudaStream_t st);
int launch_composite_backward(int64_t m, const double *means2d, const double *conics,
                              const double *colors, const double *alphas,
                              const int32_t *entry_splat, const int64_t *tile_starts,
                              const ViewParams &vp, const double *final_t,
                              const int32_t *last_contrib, const double *grad_image,
                              double *entry_grads, cudaStream_t st);
int launch_stage1(int64_t n, const double *mu_p, const double *mu_d, const double *adjust,
                  const double *prec, double px, double py, double pz, double *view,
                  double *mean_adj, double *quad, uint8_t *stage, cudaStream_t st);
int launch_stage2(int64_t n, const double *view, const double *mean_adj, const double *sh,
                  const double *sigma_prime, const double *rot, double px, double py, double pz,
                  double znear, double zfar, double f, double ox, double oy, double lim_x,
                  double lim_y, double width, double height, double low_pass, double sh_c0,
                  double sh_c1, double *means2d, double *conics, double *colors, double *depths,
                  int32_t *radii, uint8_t *stage, cudaStream_t st);

int sort_passes(int tiles);   // 8-bit LSD passes over (tile << 32 | depth32)

}  // namespace g6r
