// g6r_api.cu -- extern "C" boundary of libg6r.so (declared in include/g6r.h).
//
// Validates arguments, carves the caller's workspace, and enqueues the stage
// kernels on the caller's stream.  Never allocates, never synchronises.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

static thread_local std::string t_err;

static int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return code;
}

static int cuda_check(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(G6R_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return G6R_OK;
}

static inline size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

struct Layout {
    size_t internal, hist, proj, clear_end, tile_starts, payload, keys0, keys1, vals0, vals1,
        sort_status, total;
    int64_t sort_tiles_cap;
};

static Layout layout(int64_t n, int64_t tiles, int64_t cap, int precision) {
    Layout L{};
    size_t o = 0;
    L.internal = o;
    o = align_up(o + kNumInternal * sizeof(int64_t));
    L.hist = o;
    o = align_up(o + kMaxPasses * kBins * sizeof(unsigned));
    L.proj = o;
    const int64_t nblk = ceil_div(n > 0 ? n : 1, kBlock);
    o = align_up(o + 4 * nblk * sizeof(unsigned long long));
    L.clear_end = o;
    L.tile_starts = o;
    o = align_up(o + (tiles + 1) * sizeof(int64_t));
    L.payload = o;
    o = align_up(o + (size_t)n * (precision ? sizeof(PayloadF64) : sizeof(PayloadF32)));
    L.keys0 = o;
    o = align_up(o + (size_t)cap * 8);
    L.keys1 = o;
    o = align_up(o + (size_t)cap * 8);
    L.vals0 = o;
    o = align_up(o + (size_t)cap * 4);
    L.vals1 = o;
    o = align_up(o + (size_t)cap * 4);
    L.sort_tiles_cap = ceil_div(cap > 0 ? cap : 1, kSortTile);
    L.sort_status = o;
    o = align_up(o + (size_t)kMaxPasses * L.sort_tiles_cap * kBins * sizeof(unsigned));
    L.total = o;
    return L;
}

static Workspace carve(void *base, const Layout &L, int64_t n, int64_t cap) {
    char *b = static_cast<char *>(base);
    Workspace w{};
    w.internal = reinterpret_cast<long long *>(b + L.internal);
    w.hist = reinterpret_cast<unsigned *>(b + L.hist);
    const int64_t nblk = ceil_div(n > 0 ? n : 1, kBlock);
    unsigned long long *p = reinterpret_cast<unsigned long long *>(b + L.proj);
    w.proj_agg_m = p;
    w.proj_agg_e = p + nblk;
    w.proj_inc_m = p + 2 * nblk;
    w.proj_inc_e = p + 3 * nblk;
    w.tile_starts = reinterpret_cast<int64_t *>(b + L.tile_starts);
    w.payload = b + L.payload;
    w.keys[0] = reinterpret_cast<unsigned long long *>(b + L.keys0);
    w.keys[1] = reinterpret_cast<unsigned long long *>(b + L.keys1);
    w.vals[0] = reinterpret_cast<unsigned *>(b + L.vals0);
    w.vals[1] = reinterpret_cast<unsigned *>(b + L.vals1);
    w.sort_status = reinterpret_cast<unsigned *>(b + L.sort_status);
    w.entry_capacity = cap;
    w.sort_tiles_cap = L.sort_tiles_cap;
    return w;
}

static int check_config(const g6r_config *cfg) {
    if (!cfg) return fail(G6R_EINVAL, "config is NULL");
    if (cfg->tile_size < 1 || cfg->tile_size > 32)
        return fail(G6R_EINVAL, "tile_size must lie in [1, 32], got %d", cfg->tile_size);
    if (cfg->precision != 0 && cfg->precision != 1)
        return fail(G6R_EINVAL, "precision must be 0 (f32) or 1 (f64), got %d", cfg->precision);
    return G6R_OK;
}

static int make_view(const g6r_camera *cam, const g6r_config *cfg, ViewParams &vp) {
    if (!cam) return fail(G6R_EINVAL, "camera is NULL");
    if (cam->width < 1 || cam->height < 1) return fail(G6R_EINVAL, "width and height must be positive");
    if (!(cam->focal > 0.0) || !std::isfinite(cam->focal)) return fail(G6R_EINVAL, "focal must be positive");
    if (int rc = check_config(cfg)) return rc;
    memset(&vp, 0, sizeof vp);
    for (int k = 0; k < 3; ++k) vp.pos[k] = cam->position[k];
    for (int k = 0; k < 9; ++k) vp.rot[k] = cam->rotation[k];
    vp.focal = cam->focal;
    vp.cx = cam->cx;
    vp.cy = cam->cy;
    vp.znear = cam->znear;
    vp.zfar = cam->zfar;
    // raster.py:264-265, same association
    vp.lim_x = 1.3 * cam->width / (2.0 * cam->focal);
    vp.lim_y = 1.3 * cam->height / (2.0 * cam->focal);
    vp.width = (double)cam->width;
    vp.height = (double)cam->height;
    vp.low_pass = cfg->low_pass;
    vp.alpha_max = cfg->alpha_max;
    vp.iw = cam->width;
    vp.ih = cam->height;
    vp.tile_size = cfg->tile_size;
    vp.tiles_x = (cam->width + cfg->tile_size - 1) / cfg->tile_size;
    vp.tiles_y = (cam->height + cfg->tile_size - 1) / cfg->tile_size;
    vp.precision = cfg->precision;
    return G6R_OK;
}

static int check_ws(const Layout &L, void *ws, size_t bytes) {
    if (!ws && L.total) return fail(G6R_EINVAL, "workspace is NULL");
    if (bytes < L.total)
        return fail(G6R_EINVAL, "workspace too small: %zu bytes given, %zu needed", bytes, L.total);
    if (reinterpret_cast<uintptr_t>(ws) & 255u) return fail(G6R_EINVAL, "workspace must be 256-byte aligned");
    return G6R_OK;
}

static int check_cap(int64_t cap) {
    if (cap < 0 || cap >= (1ll << 30))
        return fail(G6R_EINVAL, "entry_capacity must lie in [0, 2^30), got %lld", (long long)cap);
    return G6R_OK;
}

}  // namespace g6r

struct g6r_profiler {
    int32_t max_views = 0, used = 0;
    cudaEvent_t *ev = nullptr;   // (max_views) x (G6R_NSTAGES + 1)
};

namespace g6r {

static void prof_mark(g6r_profiler *p, int k, cudaStream_t st) {
    if (p && p->used < p->max_views) cudaEventRecord(p->ev[p->used * (G6R_NSTAGES + 1) + k], st);
}

constexpr int kMaxSlots = 8;

// Side streams for concurrent views, created once per device and reused.
static int side_streams(int n, cudaStream_t *out) {
    static std::mutex mu;
    static std::map<int, std::vector<cudaStream_t>> pool;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    std::vector<cudaStream_t> &v = pool[dev];
    while ((int)v.size() < n) {
        cudaStream_t s;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_check("cudaStreamCreate");
        v.push_back(s);
    }
    for (int i = 0; i < n; ++i) out[i] = v[i];
    return G6R_OK;
}

static int render_one(const g6r_scene *scene, uint32_t mask, const g6r_camera *cam,
                      const g6r_config *cfg, void *ws_base, size_t ws_bytes, int64_t cap,
                      const g6r_frame *fr, const g6r_splat_out *splats, cudaStream_t st,
                      g6r_profiler *prof = nullptr) {
    if (!scene || scene->n < 0) return fail(G6R_EINVAL, "scene is NULL or has negative size");
    if (scene->n > 0 && (!scene->records || !scene->flags)) return fail(G6R_EINVAL, "scene arrays are NULL");
    if (!fr || !fr->image || !fr->counters)
        return fail(G6R_EINVAL, "frame outputs image/counters are required");
    if (int rc = check_cap(cap)) return rc;
    ViewParams vp;
    if (int rc = make_view(cam, cfg, vp)) return rc;
    const int64_t tiles = (int64_t)vp.tiles_x * vp.tiles_y;
    const Layout L = layout(scene->n, tiles, cap, vp.precision);
    if (int rc = check_ws(L, ws_base, ws_bytes)) return rc;
    Workspace ws = carve(ws_base, L, scene->n, cap);
    if (cudaMemsetAsync(ws_base, 0, L.clear_end, st) != cudaSuccess ||
        cudaMemsetAsync(fr->counters, 0, G6R_NCOUNTERS * sizeof(int64_t), st) != cudaSuccess)
        return cuda_check("memset");
    prof_mark(prof, 0, st);
    int rc = launch_project(*scene, mask, vp, ws, fr->counters, splats, true, st);
    if (rc) return cuda_check("project");
    prof_mark(prof, 1, st);
    rc = launch_sort(vp, ws, fr->counters, st);
    if (rc) return cuda_check("sort");
    prof_mark(prof, 2, st);
    rc = launch_ranges(vp, ws, fr->counters, fr->tile_starts, fr->entry_splat, st);
    if (rc) return cuda_check("ranges");
    prof_mark(prof, 3, st);
    rc = launch_composite(vp, ws.payload, ws.vals[0], ws.vals[1], ws.internal, ws.tile_starts, fr->image, fr->final_t,
                          fr->last_contrib, st);
    if (rc) return cuda_check("composite");
    prof_mark(prof, 4, st);
    if (prof && prof->used < prof->max_views) ++prof->used;
    return G6R_OK;
}

}  // namespace g6r

using namespace g6r;

extern "C" {

const char *g6r_version(void) { return "g6r 0.1.0 sm_100a"; }

const char *g6r_last_error(void) { return t_err.c_str(); }

size_t g6r_records_bytes(int64_t n) { return (size_t)(n > 0 ? n : 0) * G6R_REC_DOUBLES * sizeof(double); }

size_t g6r_workspace_bytes(int64_t n, int64_t tiles, int64_t entry_capacity, int32_t precision) {
    return layout(n, tiles, entry_capacity, precision).total;
}

int g6r_prepare(int64_t n, const double *mu_p, const double *mu_d, const double *cov_raw,
                const double *sh, const double *opacity_raw, const uint8_t *labels,
                const double *spatial_scale, double directional_scale, int32_t w_mode,
                double *records, uint8_t *flags, int64_t *label_counts, g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "n must be >= 0");
    if (w_mode != 0 && w_mode != 1) return fail(G6R_EINVAL, "w_mode must be 0 (peak) or 1 (raw)");
    if (!spatial_scale || !label_counts) return fail(G6R_EINVAL, "spatial_scale/label_counts are required");
    if (n > 0 && (!mu_p || !mu_d || !cov_raw || !sh || !opacity_raw || !labels || !records || !flags))
        return fail(G6R_EINVAL, "NULL scene array");
    if (launch_prepare(n, mu_p, mu_d, cov_raw, sh, opacity_raw, labels, spatial_scale,
                       directional_scale, w_mode, records, flags, label_counts, (cudaStream_t)stream))
        return cuda_check("prepare");
    return G6R_OK;
}

int g6r_pack_records(int64_t n, const double *mu_p, const double *mu_d, const double *sh,
                     const double *opacity, const double *w_norm, const double *adjust,
                     const double *precision_dd, const double *sigma_prime,
                     const uint8_t *degenerate, const uint8_t *labels, double *records,
                     uint8_t *flags, g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "n must be >= 0");
    if (launch_pack_records(n, mu_p, mu_d, sh, opacity, w_norm, adjust, precision_dd, sigma_prime,
                            degenerate, labels, records, flags, (cudaStream_t)stream))
        return cuda_check("pack_records");
    return G6R_OK;
}

int g6r_render(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
               const g6r_config *cfg, void *workspace, size_t workspace_bytes,
               int64_t entry_capacity, const g6r_frame *frame, const g6r_splat_out *splats,
               g6r_stream_t stream) {
    return render_one(scene, group_mask, cam, cfg, workspace, workspace_bytes, entry_capacity,
                      frame, splats, (cudaStream_t)stream);
}

int g6r_render_views(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cams,
                     int32_t count, const g6r_config *cfg, void *workspace,
                     size_t workspace_bytes, int64_t entry_capacity, const g6r_frame *frames,
                     int32_t concurrency, g6r_profiler *prof, g6r_stream_t stream) {
    if (count < 0 || (count > 0 && (!cams || !frames))) return fail(G6R_EINVAL, "bad view list");
    if (count == 0) return G6R_OK;
    if (!scene || !cfg) return fail(G6R_EINVAL, "scene/config is NULL");
    if (int rc = check_config(cfg)) return rc;
    int slots = concurrency < 1 ? 1 : (concurrency > kMaxSlots ? kMaxSlots : concurrency);
    if (slots > count) slots = count;
    const int64_t tiles = (int64_t)((cams[0].width + cfg->tile_size - 1) / cfg->tile_size) *
                          ((cams[0].height + cfg->tile_size - 1) / cfg->tile_size);
    const size_t per = layout(scene->n, tiles, entry_capacity, cfg->precision).total;
    if (workspace_bytes < per * slots)
        return fail(G6R_EINVAL, "workspace too small for %d concurrent views: %zu < %zu", slots,
                    workspace_bytes, per * slots);
    cudaStream_t main = (cudaStream_t)stream;
    if (slots == 1) {
        for (int32_t k = 0; k < count; ++k) {
            const int rc = render_one(scene, group_mask, &cams[k], cfg, workspace, per,
                                      entry_capacity, &frames[k], nullptr, main, prof);
            if (rc) return rc;
        }
        return G6R_OK;
    }
    // Views are independent: spread them over `slots` side streams, each with
    // its own workspace slice, so one view's long tile runs overlap the next
    // view's projection and sort instead of idling the other SMs.
    cudaStream_t side[kMaxSlots];
    if (int rc = side_streams(slots, side)) return rc;
    cudaEvent_t fork;
    if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) return cuda_check("event");
    cudaEventRecord(fork, main);
    for (int s = 0; s < slots; ++s) cudaStreamWaitEvent(side[s], fork, 0);
    cudaEventDestroy(fork);
    int rc = G6R_OK;
    for (int32_t k = 0; k < count && rc == G6R_OK; ++k) {
        const int s = k % slots;
        rc = render_one(scene, group_mask, &cams[k], cfg, static_cast<char *>(workspace) + per * s,
                        per, entry_capacity, &frames[k], nullptr, side[s], prof);
    }
    for (int s = 0; s < slots; ++s) {   // join (also on error, so the streams stay ordered)
        cudaEvent_t j;
        if (cudaEventCreateWithFlags(&j, cudaEventDisableTiming) == cudaSuccess) {
            cudaEventRecord(j, side[s]);
            cudaStreamWaitEvent(main, j, 0);
            cudaEventDestroy(j);
        }
    }
    return rc;
}

g6r_profiler *g6r_profiler_create(int32_t max_views) {
    if (max_views <= 0) return nullptr;
    g6r_profiler *p = new g6r_profiler;
    p->max_views = max_views;
    const int ne = max_views * (G6R_NSTAGES + 1);
    p->ev = new cudaEvent_t[ne];
    for (int k = 0; k < ne; ++k) {
        if (cudaEventCreate(&p->ev[k]) != cudaSuccess) {
            for (int j = 0; j < k; ++j) cudaEventDestroy(p->ev[j]);
            delete[] p->ev;
            delete p;
            fail(G6R_ECUDA, "cudaEventCreate failed");
            return nullptr;
        }
    }
    return p;
}

void g6r_profiler_destroy(g6r_profiler *p) {
    if (!p) return;
    for (int k = 0; k < p->max_views * (G6R_NSTAGES + 1); ++k) cudaEventDestroy(p->ev[k]);
    delete[] p->ev;
    delete p;
}

void g6r_profiler_reset(g6r_profiler *p) {
    if (p) p->used = 0;
}

int g6r_profiler_read(g6r_profiler *p, double *stage_ms, int32_t *views) {
    if (!p || !stage_ms || !views) return fail(G6R_EINVAL, "NULL profiler argument");
    for (int s = 0; s < G6R_NSTAGES; ++s) stage_ms[s] = 0.0;
    *views = p->used;
    if (!p->used) return G6R_OK;
    if (cudaEventSynchronize(p->ev[p->used * (G6R_NSTAGES + 1) - 1]) != cudaSuccess)
        return cuda_check("profiler sync");
    for (int v = 0; v < p->used; ++v)
        for (int s = 0; s < G6R_NSTAGES; ++s) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p->ev[v * (G6R_NSTAGES + 1) + s], p->ev[v * (G6R_NSTAGES + 1) + s + 1]);
            stage_ms[s] += ms;
        }
    return cuda_check("profiler read");
}

int g6r_debug_expf(int64_t n, const float *x, float *y, g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "n must be >= 0");
    if (launch_debug_expf(n, x, y, (cudaStream_t)stream)) return cuda_check("debug_expf");
    return G6R_OK;
}

int g6r_project(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
                const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                int64_t *counters, const g6r_splat_out *splats, g6r_stream_t stream) {
    if (!scene || scene->n < 0) return fail(G6R_EINVAL, "scene is NULL");
    if (!counters) return fail(G6R_EINVAL, "counters are required");
    ViewParams vp;
    if (int rc = make_view(cam, cfg, vp)) return rc;
    const Layout L = layout(scene->n, (int64_t)vp.tiles_x * vp.tiles_y, 0, vp.precision);
    if (int rc = check_ws(L, workspace, workspace_bytes)) return rc;
    Workspace ws = carve(workspace, L, scene->n, 0);
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(workspace, 0, L.clear_end, st) != cudaSuccess ||
        cudaMemsetAsync(counters, 0, G6R_NCOUNTERS * sizeof(int64_t), st) != cudaSuccess)
        return cuda_check("memset");
    if (launch_project(*scene, group_mask, vp, ws, counters, splats, false, st)) return cuda_check("project");
    return G6R_OK;
}

int g6r_bin(int64_t m, const double *means2d, const int32_t *radii, const double *depths,
            int32_t width, int32_t height, int32_t tile_size, void *workspace,
            size_t workspace_bytes, int64_t entry_capacity, int32_t *entry_splat,
            int64_t *tile_starts, int64_t *counters, g6r_stream_t stream) {
    if (m < 0) return fail(G6R_EINVAL, "m must be >= 0");
    if (m > 0 && (!means2d || !radii || !depths)) return fail(G6R_EINVAL, "NULL splat array");
    if (!counters || !tile_starts) return fail(G6R_EINVAL, "counters/tile_starts are required");
    if (int rc = check_cap(entry_capacity)) return rc;
    if (width < 1 || height < 1) return fail(G6R_EINVAL, "width and height must be positive");
    if (tile_size < 1) return fail(G6R_EINVAL, "tile_size must be positive");
    ViewParams vp{};
    vp.iw = width;
    vp.ih = height;
    vp.tile_size = tile_size;
    vp.tiles_x = (width + tile_size - 1) / tile_size;
    vp.tiles_y = (height + tile_size - 1) / tile_size;
    const Layout L = layout(m, (int64_t)vp.tiles_x * vp.tiles_y, entry_capacity, 0);
    if (int rc = check_ws(L, workspace, workspace_bytes)) return rc;
    Workspace ws = carve(workspace, L, m, entry_capacity);
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(workspace, 0, L.clear_end, st) != cudaSuccess ||
        cudaMemsetAsync(counters, 0, G6R_NCOUNTERS * sizeof(int64_t), st) != cudaSuccess)
        return cuda_check("memset");
    if (launch_duplicate(m, means2d, radii, depths, vp, ws, counters, st)) return cuda_check("duplicate");
    int final_buf = 0;
    if (launch_sort(vp, ws, counters, st)) return cuda_check("sort");
    if (launch_ranges(vp, ws, counters, tile_starts, entry_splat, st)) return cuda_check("ranges");
    return G6R_OK;
}

int g6r_composite(int64_t m, int32_t precision, const void *means2d, const void *conics,
                  const void *colors, const void *alphas, const int32_t *entry_splat,
                  const int64_t *tile_starts, int32_t tiles_x, int32_t tiles_y, int32_t tile_size,
                  int32_t width, int32_t height, void *workspace, size_t workspace_bytes,
                  void *image, void *final_t, int32_t *last_contrib, g6r_stream_t stream) {
    if (m < 0) return fail(G6R_EINVAL, "m must be >= 0");
    if (precision != 0 && precision != 1) return fail(G6R_EINVAL, "precision must be 0 or 1");
    if (tile_size < 1 || tile_size > 32) return fail(G6R_EINVAL, "tile_size must lie in [1, 32]");
    if (tiles_x != (width + tile_size - 1) / tile_size || tiles_y != (height + tile_size - 1) / tile_size)
        return fail(G6R_EINVAL, "tiles_x/tiles_y do not match width/height/tile_size");
    if (!image || !final_t || !last_contrib || !tile_starts) return fail(G6R_EINVAL, "NULL output");
    const Layout L = layout(m, (int64_t)tiles_x * tiles_y, 0, precision);
    if (int rc = check_ws(L, workspace, workspace_bytes)) return rc;
    Workspace ws = carve(workspace, L, m, 0);
    cudaStream_t st = (cudaStream_t)stream;
    if (launch_pack_payload(m, precision, means2d, conics, colors, alphas, ws.payload, st))
        return cuda_check("pack_payload");
    ViewParams vp{};
    vp.iw = width;
    vp.ih = height;
    vp.tile_size = tile_size;
    vp.tiles_x = tiles_x;
    vp.tiles_y = tiles_y;
    vp.precision = precision;
    if (launch_composite(vp, ws.payload, reinterpret_cast<const unsigned *>(entry_splat), nullptr, nullptr, tile_starts,
                         image, final_t, last_contrib, st))
        return cuda_check("composite");
    return G6R_OK;
}

int g6r_project_stage1(int64_t n, const double *mu_p, const double *mu_d, const double *adjust,
                       const double *precision_dd, double px, double py, double pz, double *view,
                       double *mean_adj, double *quad, uint8_t *stage, g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "n must be >= 0");
    if (launch_stage1(n, mu_p, mu_d, adjust, precision_dd, px, py, pz, view, mean_adj, quad, stage,
                      (cudaStream_t)stream))
        return cuda_check("stage1");
    return G6R_OK;
}

int g6r_project_stage2(int64_t n, const double *view, const double *mean_adj, const double *sh,
                       const double *sigma_prime, const double *rot, double px, double py,
                       double pz, double znear, double zfar, double f, double ox, double oy,
                       double lim_x, double lim_y, double width, double height, double low_pass,
                       double sh_c0, double sh_c1, double *means2d, double *conics,
                       double *colors, double *depths, int32_t *radii, uint8_t *stage,
                       g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "n must be >= 0");
    if (!rot) return fail(G6R_EINVAL, "rot is NULL");
    if (launch_stage2(n, view, mean_adj, sh, sigma_prime, rot, px, py, pz, znear, zfar, f, ox, oy,
                      lim_x, lim_y, width, height, low_pass, sh_c0, sh_c1, means2d, conics, colors,
                      depths, radii, stage, (cudaStream_t)stream))
        return cuda_check("stage2");
    return G6R_OK;
}

int g6r_composite_backward(int64_t m, const double *means2d, const double *conics,
                           const double *colors, const double *alphas, const int32_t *entry_splat,
                           const int64_t *tile_starts, int32_t tiles_x, int32_t tiles_y,
                           int32_t tile_size, int32_t width, int32_t height, const double *final_t,
                           const int32_t *last_contrib, const double *grad_image,
                           double *entry_grads, g6r_stream_t stream) {
    if (tile_size < 1 || tile_size > 32) return fail(G6R_EINVAL, "tile_size must lie in [1, 32]");
    ViewParams vp{};
    vp.iw = width;
    vp.ih = height;
    vp.tile_size = tile_size;
    vp.tiles_x = tiles_x;
    vp.tiles_y = tiles_y;
    vp.precision = 1;
    if (launch_composite_backward(m, means2d, conics, colors, alphas, entry_splat, tile_starts, vp,
                                  final_t, last_contrib, grad_image, entry_grads,
                                  (cudaStream_t)stream))
        return cuda_check("composite_backward");
    return G6R_OK;
}

}  // extern "C"
