// g6r_internal.h -- host-side launchers shared between the .cu translation units.
//
// Every per-view stage is launched for a *batch* of up to kMaxBatch views of
// one scene at once (grid = work x views): a launch then always has enough
// CTAs to fill the machine, a view's long tile runs overlap other views' work
// inside one kernel instead of across streams, and the projection's record
// stream is shared by the batch through L2.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/g6r.h"

namespace g6r {

constexpr int kMaxBatch = 16;

// Workspace carve-up for one view (see g6r_api.cu::layout).
struct Workspace {
    long long *internal;            // kNumInternal int64 (tickets, depth extrema, passes)
    unsigned long long *proj_status;   // look-back words, one per projection CTA
    void *payload;                  // n compositing payloads (f32 or f64)
    unsigned long long *keys[2];    // entry keys, ping-pong
    unsigned *vals[2];              // entry values (splat index), ping-pong
    unsigned *hist;                 // kMaxPasses x kBins digit totals
    unsigned *sort_counts;          // kMaxPasses x tiles_cap x kBins per-tile digit counts
    int64_t *tile_starts;           // T+1 (internal copy)
    int4 *splat_rect;               // optional (backward): per splat (entry offset, x0, y0, wx)
    uint2 *rect;                    // splat-sort path: per scene row (x0 | y0 << 16, wx | hy << 16)
    uint2 *crect;                   // splat-sort path: the tiles of rect the compositor's cull box
                                    // touches (runs without exports skip the other entries)
    unsigned *chunk_hist;           // splat-sort path: per chunk of sorted splats, T tile counts
    unsigned *warp_prefix;          // splat-sort path: per chunk, per scatter warp, packed u16 tile offsets
    unsigned *tile_total;           // splat-sort path: T entry counts
    unsigned *sched;                // T: compositor work items, longest run first (k_sched_order)
    unsigned *done_flag;            // view-complete flag (not cleared per view; reset per call)
    int64_t entry_capacity;
    int64_t sort_tiles_cap;
    int64_t nrows;                  // payload rows (scene rows, or external splats)
};

// Splat-level sort (g6r_tiles.cu): the hot-path projection writes one depth key
// and one tile rect per scene row; the rows are radix-sorted by depth and then
// expanded into tile runs by an order-preserving partition in chunks of
// kChunkSplats sorted splats.
constexpr int kChunkSplats = 2048;
// chunk size by tile-grid size: larger grids use larger chunks so the per-chunk
// work that scales with the tile count stays small per splat
__host__ __device__ inline int chunk_splats(int64_t tiles) {
    return tiles <= 1024 ? kChunkSplats : 4 * kChunkSplats;
}
constexpr int kMaxSplatSortTiles = 4096;   // larger tile grids use the entry sort
constexpr int kScatterWarps = 8;           // warps (slices) per partition chunk

struct ViewParams {
    double pos[3];
    double rot[9];
    double focal, cx, cy, znear, zfar, lim_x, lim_y, width, height;
    double low_pass, alpha_max;
    int32_t iw, ih, tile_size, tiles_x, tiles_y, precision, exp_mode;
};

struct ViewOut {
    void *image;
    void *final_t;           // may be NULL
    int32_t *last_contrib;   // may be NULL
    int64_t *counters;       // G6R_NCOUNTERS
    int32_t *entry_splat;    // optional copy of the sorted runs
    int64_t *tile_starts;    // optional copy of the tile ranges
    uint8_t *rgba8;          // optional served frame (composite over bg, quantised)
    double bg[3];
    unsigned *done_flag;     // when set: the compositor's last CTA of the view stores done_value
    unsigned done_value;
};

// One launch's views.  All views share tile size, precision and image size.
struct Batch {
    int nviews;
    int signal;   // some view has done_flag: completion signalling + view-major compositor order
    ViewParams vp[kMaxBatch];
    Workspace ws[kMaxBatch];
    ViewOut out[kMaxBatch];
};

int launch_prepare(int64_t n, const double *mu_p, const double *mu_d, const double *cov_raw,
                   const double *sh, const double *opacity_raw, const uint8_t *labels,
                   const double *ss, double ds, int w_mode, double *records, uint8_t *flags,
                   int64_t *label_counts, cudaStream_t st);
int launch_decode_records(int64_t n, const void *recs, double *mu_p, double *mu_d, double *cov_raw,
                          double *sh, double *opacity_raw, uint8_t *labels, int32_t *bad,
                          cudaStream_t st);
int launch_pack_records(int64_t n, const double *mu_p, const double *mu_d, const double *sh,
                        const double *opacity, const double *w_norm, const double *adjust,
                        const double *prec, const double *sigma_prime, const uint8_t *degenerate,
                        const uint8_t *labels, double *records, uint8_t *flags, cudaStream_t st);

// zero every view's per-view scratch region (first clear_bytes of each workspace)
// and its counters
int launch_clear(const Batch &b, size_t clear_bytes, cudaStream_t st);
// fused slice+project+compact+duplicate; writes counters[M,E,fate,overflow].
// splats (SplatBatch-shaped outputs) only for single-view batches.
int launch_project(const g6r_scene &scene, uint32_t mask, const Batch &b,
                   const g6r_splat_out *splats, bool write_entries, cudaStream_t st);
// binning of external splats (count, scan, duplicate) into ws.keys[0]/vals[0] (one view)
int launch_duplicate(int64_t m, const double *means2d, const int32_t *radii, const double *depths,
                     const Batch &b, cudaStream_t st);
// radix sort of every view's ws.keys[0]/vals[0] (E read from its counters)
// max_val: largest entry value (splat index) the views can carry
int launch_sort(const Batch &b, int64_t max_val, cudaStream_t st);
// per-tile ranges into ws.tile_starts (+ optional copies of starts / entry_splat)
int launch_ranges(const Batch &b, int64_t max_val, cudaStream_t st);
// Which projection/sort a render uses: ordered (compacted SplatBatch outputs,
// entry sort) when splat outputs or per-splat rects are requested; otherwise
// the splat-level sort when the tile grid fits kMaxSplatSortTiles.
bool projection_ordered(const Batch &b, const g6r_splat_out *splats, bool write_entries);
bool splat_sort_applies(const Batch &b);
// splat-level sort + tile partition (hot path); n = scene rows
int launch_splat_sort(const Batch &b, int64_t n, cudaStream_t st);
int launch_tile_partition(const Batch &b, int64_t n, int vbits, cudaStream_t st);
int launch_debug_expf(int64_t n, const float *x, float *y, cudaStream_t st);
int launch_debug_exp(int64_t n, const double *x, double *y, cudaStream_t st);
int launch_pack_payload(int64_t m, int precision, const void *means2d, const void *conics,
                        const void *colors, const void *alphas, void *payload, cudaStream_t st);
// sorted: entry values are the view's sorted ping-pong buffer; otherwise vals[0] holds them
int launch_composite(const Batch &b, bool sorted, cudaStream_t st);
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

int launch_backward(const ViewParams &vp, const g6r_scene &scene, const Workspace &ws,
                    int64_t *counters, const double *final_t, const int32_t *last,
                    const double *grad_image, const int64_t *gids, uint8_t *drawn, double *egrad, double *gsplat,
                    const double *mu_p, const double *mu_d, const double *cov_raw, const double *sh,
                    const double *ss, double ds, int w_mode, double *g_mu_p, double *g_mu_d,
                    double *g_cov_raw, double *g_sh, double *g_opacity_raw, cudaStream_t st);

int sort_passes(int tiles);   // upper bound on radix passes for `tiles` tiles

// Launch trace (G6R_TRACE=1 in the environment): a CUDA event is recorded on
// the stream after every kernel launch, labelled with the kernel; the C ABI's
// g6r_trace_dump prints per-launch device intervals.  Off by default (one
// branch per launch).
void trace_mark(const char *label, cudaStream_t st);

// scene ingest (g6r_ingest.cu)
struct DecodeArgsHost {
    const void *psi;
    int psi_f32;
    const double *base;
    const uint8_t *lab;
    int64_t V;
    int dh, dw;
    double spacing[3], origin[3], dir[9];
    double *mu_p, *mu_d, *cov_raw, *sh, *opacity_raw;
    uint8_t *labels;
};
size_t compact_workspace_bytes(int64_t n);
int launch_decode_count(int64_t V, const uint8_t *lab, void *ws, int64_t *count, cudaStream_t st);
int launch_decode_emit(const DecodeArgsHost &h, void *ws, cudaStream_t st);
int launch_filter_rows(int64_t n, const uint8_t *lab, uint32_t mask, const double *const in[5],
                       double *const out[5], uint8_t *labels, void *ws, int64_t *count,
                       cudaStream_t st);

// fine-tune loop (g6r_train.cu)
size_t loss_workspace_bytes(int h, int w);
int loss_grad(const double *pred, const double *tgt, int tc, int h, int w, double lambda_l1,
              double lambda_ssim, int scales, const double *weights, void *ws, double *grad,
              double *parts, cudaStream_t st);
int adam_step(int64_t n, double *p, const double *g, double *m, double *v, double lr, double bias1,
              double bias2, cudaStream_t st);
int nonfinite(int64_t n, const double *x, int32_t *flag, cudaStream_t st);

}  // namespace g6r
