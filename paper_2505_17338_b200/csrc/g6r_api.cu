// g6r_api.cu -- extern "C" boundary of libg6r.so (declared in include/g6r.h).
//
// Validates arguments, carves the caller's workspace, and enqueues the stage
// kernels on the caller's stream.  Never allocates device memory, never
// synchronises (except g6r_profiler_read, which waits on its own events).
// Views are rendered in batches: every stage kernel takes up to kMaxBatch views
// per launch (grid = work x views).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

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
        sort_counts, rect, crect, chunk_hist, warp_prefix, tile_total, sched, done, total;
    int64_t sort_tiles_cap, nrows;
};

// Per-view workspace layout.  [0, clear_end) is zeroed before every view.
static Layout layout(int64_t n, int64_t tiles, int64_t cap, int precision) {
    Layout L{};
    size_t o = 0;
    L.internal = o;
    o = align_up(o + kNumInternal * sizeof(int64_t));
    L.hist = o;
    o = align_up(o + kMaxPasses * kBins * sizeof(unsigned));
    L.proj = o;
    const int64_t nblk = ceil_div(n > 0 ? n : 1, kBlock);
    o = align_up(o + nblk * sizeof(unsigned long long));
    L.clear_end = o;
    L.tile_starts = o;
    o = align_up(o + (tiles + 1) * sizeof(int64_t));
    L.payload = o;
    o = align_up(o + (size_t)n * (precision ? sizeof(PayloadF64) : sizeof(PayloadF32)));
    // the sort buffers hold either the E tile entries or the n splat keys
    const int64_t items = std::max<int64_t>(cap, n);
    L.keys0 = o;
    o = align_up(o + (size_t)items * 8);
    L.keys1 = o;
    o = align_up(o + (size_t)items * 8);
    L.vals0 = o;
    o = align_up(o + (size_t)cap * 4);
    L.vals1 = o;
    o = align_up(o + (size_t)cap * 4);
    L.sort_tiles_cap = ceil_div(items > 0 ? items : 1, kSortTile);
    L.sort_counts = o;
    o = align_up(o + (size_t)kMaxPasses * L.sort_tiles_cap * kBins * sizeof(unsigned));
    L.rect = o;
    o = align_up(o + (size_t)n * sizeof(uint2));
    L.crect = o;
    o = align_up(o + (size_t)n * sizeof(uint2));
    L.chunk_hist = o;
    o = align_up(o + (size_t)ceil_div(n > 0 ? n : 1, chunk_splats(tiles)) * tiles * sizeof(unsigned));
    L.warp_prefix = o;   // kScatterWarps x ceil(T/2) packed words per chunk
    o = align_up(o + (size_t)ceil_div(n > 0 ? n : 1, chunk_splats(tiles)) * kScatterWarps * ((tiles + 1) / 2) *
                         sizeof(unsigned));
    L.tile_total = o;
    o = align_up(o + (size_t)tiles * sizeof(unsigned));
    L.sched = o;   // compositor work order (this view's slice of the batch's ranking)
    o = align_up(o + (size_t)tiles * sizeof(unsigned));
    L.done = o;    // view-complete flag (reset once per call, not per view)
    o = align_up(o + sizeof(unsigned));
    L.total = o;
    L.nrows = n;
    return L;
}

static Workspace carve(void *base, const Layout &L, int64_t cap) {
    char *b = static_cast<char *>(base);
    Workspace w{};
    w.internal = reinterpret_cast<long long *>(b + L.internal);
    w.hist = reinterpret_cast<unsigned *>(b + L.hist);
    w.proj_status = reinterpret_cast<unsigned long long *>(b + L.proj);
    w.tile_starts = reinterpret_cast<int64_t *>(b + L.tile_starts);
    w.payload = b + L.payload;
    w.keys[0] = reinterpret_cast<unsigned long long *>(b + L.keys0);
    w.keys[1] = reinterpret_cast<unsigned long long *>(b + L.keys1);
    w.vals[0] = reinterpret_cast<unsigned *>(b + L.vals0);
    w.vals[1] = reinterpret_cast<unsigned *>(b + L.vals1);
    w.sort_counts = reinterpret_cast<unsigned *>(b + L.sort_counts);
    w.rect = reinterpret_cast<uint2 *>(b + L.rect);
    w.crect = reinterpret_cast<uint2 *>(b + L.crect);
    w.chunk_hist = reinterpret_cast<unsigned *>(b + L.chunk_hist);
    w.warp_prefix = reinterpret_cast<unsigned *>(b + L.warp_prefix);
    w.tile_total = reinterpret_cast<unsigned *>(b + L.tile_total);
    w.sched = reinterpret_cast<unsigned *>(b + L.sched);
    w.done_flag = reinterpret_cast<unsigned *>(b + L.done);
    w.entry_capacity = cap;
    w.sort_tiles_cap = L.sort_tiles_cap;
    w.nrows = L.nrows;
    return w;
}

static int check_config(const g6r_config *cfg) {
    if (!cfg) return fail(G6R_EINVAL, "config is NULL");
    if (cfg->tile_size < 1 || cfg->tile_size > 32)
        return fail(G6R_EINVAL, "tile_size must lie in [1, 32], got %d", cfg->tile_size);
    if (cfg->precision != 0 && cfg->precision != 1)
        return fail(G6R_EINVAL, "precision must be 0 (f32) or 1 (f64), got %d", cfg->precision);
    if (cfg->exp_mode != 0 && cfg->exp_mode != 1)
        return fail(G6R_EINVAL, "exp_mode must be 0 (exact) or 1 (fast), got %d", cfg->exp_mode);
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
    vp.exp_mode = cfg->exp_mode;
    return G6R_OK;
}

static int check_ws(size_t need, void *ws, size_t bytes) {
    if (!ws && need) return fail(G6R_EINVAL, "workspace is NULL");
    if (bytes < need)
        return fail(G6R_EINVAL, "workspace too small: %zu bytes given, %zu needed", bytes, need);
    if (reinterpret_cast<uintptr_t>(ws) & 255u) return fail(G6R_EINVAL, "workspace must be 256-byte aligned");
    return G6R_OK;
}

static int check_cap(int64_t cap) {
    if (cap < 0 || cap >= (1ll << 30))
        return fail(G6R_EINVAL, "entry_capacity must lie in [0, 2^30), got %lld", (long long)cap);
    return G6R_OK;
}

// zero the batch's per-view scratch heads and counters in one launch
__global__ void k_clear(const __grid_constant__ Batch b, size_t clear_words) {
    const int v = blockIdx.y;
    unsigned long long *w = reinterpret_cast<unsigned long long *>(b.ws[v].internal);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < clear_words;
         i += (size_t)gridDim.x * blockDim.x)
        w[i] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x < G6R_NCOUNTERS) b.out[v].counters[threadIdx.x] = 0;
}

int launch_clear(const Batch &b, size_t clear_bytes, cudaStream_t st) {
    const size_t words = clear_bytes / 8;
    const unsigned gx = (unsigned)std::max<size_t>(1, std::min<size_t>((words + 255) / 256, 64));
    k_clear<<<dim3(gx, b.nviews), 256, 0, st>>>(b, words);
    trace_mark("clear", st);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

// --- launch trace -----------------------------------------------------------
struct TraceRec {
    const char *label;
    cudaEvent_t ev;
};
static std::mutex g_trace_mu;
static std::vector<TraceRec> g_trace;
static int g_trace_on = -1;

static bool trace_enabled() {
    if (g_trace_on < 0) {
        const char *e = getenv("G6R_TRACE");
        g_trace_on = (e && e[0] == '1') ? 1 : 0;
    }
    return g_trace_on == 1;
}

void trace_mark(const char *label, cudaStream_t st) {
    if (!trace_enabled()) return;
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) != cudaSuccess) return;
    cudaEventRecord(ev, st);
    std::lock_guard<std::mutex> lock(g_trace_mu);
    g_trace.push_back(TraceRec{label, ev});
}

}  // namespace g6r

struct g6r_profiler {
    int32_t max_batches = 0, used = 0, views = 0;
    cudaEvent_t *ev = nullptr;   // (max_batches) x (G6R_NSTAGES + 1)
    int32_t *nv = nullptr;       // views per recorded batch
};

namespace g6r {

// --- host copies gated by view completion (g6r_frame.host_image / host_rgba8)
// cuStreamWaitValue32 (driver entry point, no libcuda link): the copy stream
// waits until the compositor's last CTA of a view has stored the batch's
// value into the view's flag, then copies that view while the rest renders.
typedef int (*WaitValue32Fn)(cudaStream_t, unsigned long long, unsigned, unsigned);
constexpr unsigned kWaitGeq = 0x0;   // CU_STREAM_WAIT_VALUE_GEQ

static WaitValue32Fn wait_value_fn() {
    static WaitValue32Fn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return reinterpret_cast<WaitValue32Fn>(p);
    }();
    return fn;
}

static cudaStream_t g_copy[64];
static std::mutex g_copy_mu;
static cudaStream_t copy_stream() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(g_copy_mu);
    if (!g_copy[dev] && cudaStreamCreateWithFlags(&g_copy[dev], cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    return g_copy[dev];
}

static bool wants_host_copy(const g6r_frame *frames, int count) {
    for (int v = 0; v < count; ++v)
        if (frames[v].host_image || frames[v].host_rgba8) return true;
    return false;
}

// zero the done flags of every view slot the call's workspace holds
__global__ void k_reset_done(char *base, size_t half_bytes, size_t view_bytes, size_t off, int lanes, int nb) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= lanes * nb) return;
    *reinterpret_cast<unsigned *>(base + (size_t)(k / nb) * half_bytes + (size_t)(k % nb) * view_bytes + off) = 0u;
}

struct CopyCtx {
    cudaStream_t cs = nullptr;   // null: no host copies in this call
    unsigned value = 0;          // batch ordinal + 1 (monotonic per flag slot in a call)
};

// Start of a call with host copies: reset the flags on `st`, order the copy
// stream after that.
static int copy_begin(CopyCtx &cc, char *ws, size_t half_bytes, size_t view_bytes, size_t off, int lanes,
                      int nb, cudaStream_t st) {
    cc.cs = copy_stream();
    if (!cc.cs) return G6R_ECUDA;
    k_reset_done<<<(unsigned)ceil_div((int64_t)lanes * nb, 128), 128, 0, st>>>(ws, half_bytes, view_bytes, off,
                                                                               lanes, nb);
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return G6R_ECUDA;
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(cc.cs, ev, 0);
    cudaEventDestroy(ev);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

static void copy_end(const CopyCtx &cc, cudaStream_t st) {
    if (!cc.cs) return;
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return;
    cudaEventRecord(ev, cc.cs);
    cudaStreamWaitEvent(st, ev, 0);
    cudaEventDestroy(ev);
}

// After a batch's compositor launch on `st`: each view's copies on the copy
// stream, gated by its flag (or, without stream memory operations, by an event
// after the batch).
static int enqueue_host_copies(const Batch &b, const g6r_frame *frames, const CopyCtx &cc, cudaStream_t st) {
    const WaitValue32Fn wait = wait_value_fn();
    bool evented = false;
    for (int v = 0; v < b.nviews; ++v) {
        const g6r_frame &f = frames[v];
        if (!f.host_image && !f.host_rgba8) continue;
        bool gated = false;
        if (wait && b.out[v].done_flag)
            gated = wait(cc.cs, (unsigned long long)(uintptr_t)b.out[v].done_flag, b.out[v].done_value, kWaitGeq) == 0;
        if (!gated && !evented) {
            cudaEvent_t ev;
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return G6R_ECUDA;
            cudaEventRecord(ev, st);
            cudaStreamWaitEvent(cc.cs, ev, 0);
            cudaEventDestroy(ev);
            evented = true;
        }
        const size_t px = (size_t)b.vp[v].iw * b.vp[v].ih;
        if (f.host_image && f.image)
            cudaMemcpyAsync(f.host_image, f.image, px * 4 * (b.vp[v].precision ? 8 : 4), cudaMemcpyDeviceToHost,
                            cc.cs);
        if (f.host_rgba8 && f.rgba8) cudaMemcpyAsync(f.host_rgba8, f.rgba8, px * 4, cudaMemcpyDeviceToHost, cc.cs);
    }
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

static void prof_mark(g6r_profiler *p, int k, cudaStream_t st) {
    if (p && p->used < p->max_batches) cudaEventRecord(p->ev[p->used * (G6R_NSTAGES + 1) + k], st);
}

// Render one batch of views (all stages, CUDA events between them when profiled).
static int render_batch(const g6r_scene *scene, uint32_t mask, const g6r_camera *cams, int nviews,
                        const g6r_config *cfg, void *ws_base, size_t ws_bytes, int64_t cap,
                        const g6r_frame *frames, const g6r_splat_out *splats, cudaStream_t st,
                        g6r_profiler *prof, const CopyCtx *cc = nullptr, cudaStream_t hp = nullptr,
                        int hp_mode = 0) {
    if (!scene || scene->n < 0) return fail(G6R_EINVAL, "scene is NULL or has negative size");
    if (scene->n > 0 && (!scene->records || !scene->flags)) return fail(G6R_EINVAL, "scene arrays are NULL");
    if (nviews < 1 || nviews > kMaxBatch) return fail(G6R_EINVAL, "batch of %d views", nviews);
    if (int rc = check_cap(cap)) return rc;
    Batch b;
    memset(&b, 0, sizeof b);
    b.nviews = nviews;
    for (int v = 0; v < nviews; ++v) {
        const g6r_frame *fr = &frames[v];
        if ((!fr->image && !fr->rgba8) || !fr->counters)
            return fail(G6R_EINVAL, "frame outputs image (or rgba8) and counters are required");
        if (int rc = make_view(&cams[v], cfg, b.vp[v])) return rc;
        if (b.vp[v].iw != b.vp[0].iw || b.vp[v].ih != b.vp[0].ih)
            return fail(G6R_EINVAL, "views of one batch must share the image size");
    }
    const int64_t tiles = (int64_t)b.vp[0].tiles_x * b.vp[0].tiles_y;
    const Layout L = layout(scene->n, tiles, cap, cfg->precision);
    if (int rc = check_ws(L.total * nviews, ws_base, ws_bytes)) return rc;
    for (int v = 0; v < nviews; ++v) {
        b.ws[v] = carve(static_cast<char *>(ws_base) + L.total * v, L, cap);
        b.out[v] = ViewOut{frames[v].image, frames[v].final_t, frames[v].last_contrib,
                           frames[v].counters, frames[v].entry_splat, frames[v].tile_starts,
                           frames[v].rgba8,
                           {frames[v].background[0], frames[v].background[1],
                            frames[v].background[2]},
                           nullptr, 0u};
        if (cc && cc->cs && (frames[v].host_image || frames[v].host_rgba8)) {
            b.out[v].done_flag = b.ws[v].done_flag;
            b.out[v].done_value = cc->value;
            b.signal = 1;
        }
    }
    // hp (pipelined batches): the pre-composite stages on a high-priority
    // stream, so their CTAs take SM slots as the other lane's compositor CTAs
    // retire instead of queueing behind them (hp_mode 2: clear, projection,
    // sort and partition; 1: sort and partition only)
    cudaStream_t st0 = st;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    auto to_hp = [&]() {
        if (cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming) != cudaSuccess) return;
        cudaEventRecord(ev_in, st0);
        cudaStreamWaitEvent(hp, ev_in, 0);
        st = hp;
    };
    if (hp && hp_mode == 2) to_hp();
    if (launch_clear(b, L.clear_end, st)) return cuda_check("clear");
    prof_mark(prof, 0, st);
    const g6r_splat_out *so = nviews == 1 ? splats : nullptr;
    const bool splat_sort = !projection_ordered(b, so, true) && splat_sort_applies(b);
    if (launch_project(*scene, mask, b, so, true, st)) return cuda_check("project");
    prof_mark(prof, 1, st);
    if (hp && hp_mode == 1) to_hp();
    if (splat_sort) {   // depth sort of the splats + order-preserving tile expansion
        if (launch_splat_sort(b, scene->n, st)) return cuda_check("sort");
        prof_mark(prof, 2, st);
        prof_mark(prof, 3, st);
    } else {            // tile entries: radix sort of (tile, depth) keys, then ranges
        if (launch_sort(b, scene->n, st)) return cuda_check("sort");
        prof_mark(prof, 2, st);
        if (launch_ranges(b, scene->n, st)) return cuda_check("ranges");
        prof_mark(prof, 3, st);
    }
    if (st != st0) {   // back to the lane stream for the compositor
        if (cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming) == cudaSuccess) {
            cudaEventRecord(ev_out, st);
            cudaStreamWaitEvent(st0, ev_out, 0);
        }
        st = st0;
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_out) cudaEventDestroy(ev_out);
    }
    if (launch_composite(b, true, st)) return cuda_check("composite");
    prof_mark(prof, 4, st);
    if (cc && cc->cs)
        if (enqueue_host_copies(b, frames, *cc, st)) return cuda_check("host copies");
    if (prof && prof->used < prof->max_batches) {
        prof->nv[prof->used++] = nviews;
        prof->views += nviews;
    }
    return G6R_OK;
}

}  // namespace g6r

using namespace g6r;

extern "C" {

const char *g6r_version(void) { return "g6r 0.2.0 sm_100a"; }

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
    if (n >= (1ll << 30)) return fail(G6R_EINVAL, "scenes are limited to 2^30 Gaussians");
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
    if (!frame) return fail(G6R_EINVAL, "frame is NULL");
    if (int rc = check_config(cfg)) return rc;
    const cudaStream_t st = (cudaStream_t)stream;
    if (!wants_host_copy(frame, 1))
        return render_batch(scene, group_mask, cam, 1, cfg, workspace, workspace_bytes, entry_capacity,
                            frame, splats, st, nullptr);
    if (!scene || !cam || cam->width < 1 || cam->height < 1 || cfg->tile_size < 1)
        return render_batch(scene, group_mask, cam, 1, cfg, workspace, workspace_bytes, entry_capacity,
                            frame, splats, st, nullptr);   // reports the argument error
    const int64_t tx = (cam->width + cfg->tile_size - 1) / cfg->tile_size;
    const int64_t ty = (cam->height + cfg->tile_size - 1) / cfg->tile_size;
    const Layout L = layout(scene->n, tx * ty, entry_capacity, cfg->precision);
    if (int rc = check_ws(L.total, workspace, workspace_bytes)) return rc;
    CopyCtx cc;
    cc.value = 1;
    if (copy_begin(cc, static_cast<char *>(workspace), L.total, L.total, L.done, 1, 1, st))
        return cuda_check("copy stream");
    const int rc = render_batch(scene, group_mask, cam, 1, cfg, workspace, workspace_bytes, entry_capacity,
                                frame, splats, st, nullptr, &cc);
    copy_end(cc, st);
    return rc;
}

// Two internal streams per device for pipelining consecutive batches: a
// batch's latency-bound projection and sort overlap the previous batch's
// issue-bound compositing.
constexpr int kMaxLanes = 4;
static cudaStream_t g_lane[64][kMaxLanes], g_lane_hp[64][kMaxLanes];
static std::mutex g_lane_mu;

static int lane_streams(cudaStream_t *out, cudaStream_t *hp) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 1;
    std::lock_guard<std::mutex> lock(g_lane_mu);
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    for (int k = 0; k < kMaxLanes; ++k) {
        if (!g_lane[dev][k] && cudaStreamCreateWithFlags(&g_lane[dev][k], cudaStreamNonBlocking) != cudaSuccess)
            return 1;
        if (!g_lane_hp[dev][k] &&
            cudaStreamCreateWithPriority(&g_lane_hp[dev][k], cudaStreamNonBlocking, greatest) != cudaSuccess)
            return 1;
        out[k] = g_lane[dev][k];
        hp[k] = g_lane_hp[dev][k];
    }
    return 0;
}

int g6r_render_views(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cams,
                     int32_t count, const g6r_config *cfg, void *workspace,
                     size_t workspace_bytes, int64_t entry_capacity, const g6r_frame *frames,
                     int32_t batch, g6r_profiler *prof, g6r_stream_t stream) {
    if (count < 0 || (count > 0 && (!cams || !frames))) return fail(G6R_EINVAL, "bad view list");
    if (count == 0) return G6R_OK;
    if (int rc = check_config(cfg)) return rc;
    if (!scene) return fail(G6R_EINVAL, "scene is NULL");
    const int nb_max = batch < 1 ? 1 : (batch > kMaxBatch ? kMaxBatch : batch);
    // balanced batches: count views in ceil(count / nb_max) launches of (almost)
    // equal size -- 20 views at 16 run as 10 + 10, not 16 + a 4-view tail whose
    // heaviest tiles bound a launch of its own
    const int nbatches = (int)((count + nb_max - 1) / nb_max);
    const int nb = (int)((count + nbatches - 1) / nbatches);
    const cudaStream_t st = (cudaStream_t)stream;
    // Pipelined when the workspace holds two batches, there are at least two
    // batches, and no profiler is attached (stage timings need one lane).
    size_t per_batch = 0;
    if (cams[0].width > 0 && cams[0].height > 0 && cfg->tile_size > 0) {
        const int64_t tx = (cams[0].width + cfg->tile_size - 1) / cfg->tile_size;
        const int64_t ty = (cams[0].height + cfg->tile_size - 1) / cfg->tile_size;
        per_batch = layout(scene->n, tx * ty, entry_capacity, cfg->precision).total * (size_t)nb;
    }
    // lanes = how many batch slices the workspace holds (2..kMaxLanes)
    const int lanes = per_batch ? (int)std::min<size_t>(kMaxLanes, workspace_bytes / per_batch) : 1;
    const bool piped = !prof && count > nb && lanes >= 2;
    // host copies: flags reset for every slot the call uses, copy stream ordered after
    CopyCtx cc;
    if (per_batch && wants_host_copy(frames, count)) {
        const int64_t tx = (cams[0].width + cfg->tile_size - 1) / cfg->tile_size;
        const int64_t ty = (cams[0].height + cfg->tile_size - 1) / cfg->tile_size;
        const Layout L = layout(scene->n, tx * ty, entry_capacity, cfg->precision);
        if (check_ws(per_batch * (piped ? lanes : 1), workspace, workspace_bytes) == G6R_OK &&
            copy_begin(cc, static_cast<char *>(workspace), per_batch, L.total, L.done, piped ? lanes : 1, nb, st))
            return cuda_check("copy stream");
    }
    if (!piped) {
        int rc = G6R_OK;
        for (int32_t k = 0, i = 0; k < count && !rc; k += nb, ++i) {
            const int nv = count - k < nb ? count - k : nb;
            cc.value = (unsigned)i + 1;
            rc = render_batch(scene, group_mask, &cams[k], nv, cfg, workspace, workspace_bytes,
                              entry_capacity, &frames[k], nullptr, st, prof, &cc);
        }
        copy_end(cc, st);
        return rc;
    }
    cudaStream_t lane[kMaxLanes], lane_hp[kMaxLanes];
    if (lane_streams(lane, lane_hp)) return cuda_check("lane streams");
    // each batch's pre-composite stages run on its lane's high-priority twin
    // stream (render_batch); G6R_PRIO=0 keeps them on the lane, 1 moves only
    // the sort (A/B probe).  Measured on the bench's 20 views: e2e 4395 -> 4443
    // views/s (5 runs each), device rate unchanged within its +-3 % spread.
    static const int hp_mode = [] {
        const char *e = getenv("G6R_PRIO");
        return e ? atoi(e) : 2;
    }();
    cudaEvent_t fork, join[kMaxLanes];
    if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) return cuda_check("event");
    cudaEventRecord(fork, st);
    for (int l = 0; l < lanes; ++l) cudaStreamWaitEvent(lane[l], fork, 0);
    int rc = G6R_OK;
    for (int32_t k = 0, i = 0; k < count && !rc; k += nb, ++i) {
        const int nv = count - k < nb ? count - k : nb;
        char *half = static_cast<char *>(workspace) + (size_t)(i % lanes) * per_batch;
        cc.value = (unsigned)i + 1;
        rc = render_batch(scene, group_mask, &cams[k], nv, cfg, half, per_batch, entry_capacity,
                          &frames[k], nullptr, lane[i % lanes], nullptr, &cc,
                          hp_mode ? lane_hp[i % lanes] : nullptr, hp_mode);
    }
    for (int l = 0; l < lanes; ++l) {   // join (also on error, so the caller's stream stays ordered)
        cudaEventCreateWithFlags(&join[l], cudaEventDisableTiming);
        cudaEventRecord(join[l], lane[l]);
        cudaStreamWaitEvent(st, join[l], 0);
        cudaEventDestroy(join[l]);
    }
    cudaEventDestroy(fork);
    copy_end(cc, st);
    return rc;
}

g6r_profiler *g6r_profiler_create(int32_t max_batches) {
    if (max_batches <= 0) return nullptr;
    g6r_profiler *p = new g6r_profiler;
    p->max_batches = max_batches;
    const int ne = max_batches * (G6R_NSTAGES + 1);
    p->ev = new cudaEvent_t[ne];
    p->nv = new int32_t[max_batches];
    for (int k = 0; k < ne; ++k) {
        if (cudaEventCreate(&p->ev[k]) != cudaSuccess) {
            for (int j = 0; j < k; ++j) cudaEventDestroy(p->ev[j]);
            delete[] p->ev;
            delete[] p->nv;
            delete p;
            fail(G6R_ECUDA, "cudaEventCreate failed");
            return nullptr;
        }
    }
    return p;
}

void g6r_profiler_destroy(g6r_profiler *p) {
    if (!p) return;
    for (int k = 0; k < p->max_batches * (G6R_NSTAGES + 1); ++k) cudaEventDestroy(p->ev[k]);
    delete[] p->ev;
    delete[] p->nv;
    delete p;
}

void g6r_profiler_reset(g6r_profiler *p) {
    if (p) p->used = p->views = 0;
}

int g6r_profiler_read(g6r_profiler *p, double *stage_ms, int32_t *views) {
    if (!p || !stage_ms || !views) return fail(G6R_EINVAL, "NULL profiler argument");
    for (int s = 0; s < G6R_NSTAGES; ++s) stage_ms[s] = 0.0;
    *views = p->views;
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

int g6r_host_device_pointer(void *host, void **device) {
    if (!host || !device) return fail(G6R_EINVAL, "host/device pointer is NULL");
    *device = nullptr;
    if (cudaHostGetDevicePointer(device, host, 0) != cudaSuccess) {
        cudaGetLastError();   // not page-locked (or not mapped): clear the sticky-free error
        *device = nullptr;
        return fail(G6R_EINVAL, "pointer is not page-locked host memory mapped for the device");
    }
    return G6R_OK;
}

int g6r_trace_dump(const char *path) {
    std::lock_guard<std::mutex> lock(g_trace_mu);
    if (g_trace.empty()) return G6R_OK;
    cudaEventSynchronize(g_trace.back().ev);
    FILE *f = path ? fopen(path, "w") : stderr;
    if (!f) return fail(G6R_EINVAL, "cannot open %s", path);
    fprintf(f, "label,ms_since_previous_mark\n");
    for (size_t i = 1; i < g_trace.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_trace[i - 1].ev, g_trace[i].ev);
        fprintf(f, "%s,%.4f\n", g_trace[i].label, ms);
    }
    if (path) fclose(f);
    for (auto &r : g_trace) cudaEventDestroy(r.ev);
    g_trace.clear();
    return cuda_check("trace dump");
}

// Backward workspace: the f64 forward layout followed by the gradient buffers.
struct BwdLayout {
    size_t fwd, gids, drawn, rect, egrad, gsplat, final_t, last, image, total;
};

static BwdLayout bwd_layout(int64_t n, int32_t width, int32_t height, int32_t tile_size, int64_t cap) {
    BwdLayout B{};
    const int64_t tiles = (int64_t)((width + tile_size - 1) / tile_size) * ((height + tile_size - 1) / tile_size);
    const int64_t hw = (int64_t)width * height;
    const int64_t nn = n > 0 ? n : 1;
    size_t o = layout(n, tiles, cap, 1).total;
    B.fwd = 0;
    B.gids = o;
    o = align_up(o + nn * 8);
    B.drawn = o;   // per scene row: drawn in this view (k_splat_grad_sum)
    o = align_up(o + nn);
    B.rect = o;
    o = align_up(o + nn * 16);
    B.egrad = o;   // one 9-double row per entry and per tile band (2)
    o = align_up(o + (size_t)(cap > 0 ? cap : 1) * 72 * 2);
    B.gsplat = o;
    o = align_up(o + nn * 72);
    B.final_t = o;
    o = align_up(o + hw * 8);
    B.last = o;
    o = align_up(o + hw * 4);
    B.image = o;
    o = align_up(o + hw * 32);
    B.total = o;
    return B;
}

size_t g6r_backward_workspace_bytes(int64_t n, int32_t width, int32_t height, int32_t tile_size,
                                    int64_t entry_capacity) {
    if (n < 0 || width < 1 || height < 1 || tile_size < 1) return 0;
    return bwd_layout(n, width, height, tile_size, entry_capacity).total;
}

// Validate and carve a backward workspace (shared by the forward-with-state
// and apply halves, which must see the same scene, camera and capacity).
static int bwd_setup(const g6r_scene *scene, const g6r_camera *cam, const g6r_config *cfg,
                     void *workspace, size_t workspace_bytes, int64_t cap, int64_t *counters,
                     double *image_out, Batch &b, BwdLayout &B) {
    if (!scene || scene->n < 0) return fail(G6R_EINVAL, "scene is NULL");
    if (int rc = check_config(cfg)) return rc;
    if (cfg->precision != 1) return fail(G6R_EINVAL, "the backward pass runs in f64 (precision=1)");
    if (cfg->tile_size != 16) return fail(G6R_EINVAL, "the backward kernel supports tile_size 16");
    if (!counters) return fail(G6R_EINVAL, "counters are required");
    if (int rc = check_cap(cap)) return rc;
    ViewParams vp;
    if (int rc = make_view(cam, cfg, vp)) return rc;
    B = bwd_layout(scene->n, vp.iw, vp.ih, vp.tile_size, cap);
    if (int rc = check_ws(B.total, workspace, workspace_bytes)) return rc;
    char *base = static_cast<char *>(workspace);
    const Layout L = layout(scene->n, (int64_t)vp.tiles_x * vp.tiles_y, cap, 1);
    memset(&b, 0, sizeof b);
    b.nviews = 1;
    b.vp[0] = vp;
    b.ws[0] = carve(base, L, cap);
    b.ws[0].splat_rect = reinterpret_cast<int4 *>(base + B.rect);
    b.out[0] = ViewOut{image_out ? (void *)image_out : (void *)(base + B.image),
                       base + B.final_t, reinterpret_cast<int32_t *>(base + B.last), counters,
                       nullptr, nullptr};
    return G6R_OK;
}

int g6r_backward_forward(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
                         const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                         int64_t entry_capacity, int64_t *counters, double *image_out,
                         g6r_stream_t stream) {
    Batch b;
    BwdLayout B;
    if (int rc = bwd_setup(scene, cam, cfg, workspace, workspace_bytes, entry_capacity, counters,
                           image_out, b, B))
        return rc;
    g6r_splat_out so{};
    so.gids = reinterpret_cast<int64_t *>(static_cast<char *>(workspace) + B.gids);
    cudaStream_t st = (cudaStream_t)stream;
    const Layout L = layout(scene->n, (int64_t)b.vp[0].tiles_x * b.vp[0].tiles_y, entry_capacity, 1);
    if (launch_clear(b, L.clear_end, st)) return cuda_check("clear");
    if (launch_project(*scene, group_mask, b, &so, true, st)) return cuda_check("project");
    if (launch_sort(b, scene->n, st)) return cuda_check("sort");
    if (launch_ranges(b, scene->n, st)) return cuda_check("ranges");
    if (launch_composite(b, true, st)) return cuda_check("composite");
    return G6R_OK;
}

int g6r_backward_apply(const g6r_scene *scene, const g6r_camera *cam, const g6r_config *cfg,
                       void *workspace, size_t workspace_bytes, int64_t entry_capacity,
                       const double *mu_p, const double *mu_d, const double *cov_raw,
                       const double *sh, const double *spatial_scale, double directional_scale,
                       int32_t w_mode, const double *grad_image, double *g_mu_p, double *g_mu_d,
                       double *g_cov_raw, double *g_sh, double *g_opacity_raw, int64_t *counters,
                       g6r_stream_t stream) {
    Batch b;
    BwdLayout B;
    if (int rc = bwd_setup(scene, cam, cfg, workspace, workspace_bytes, entry_capacity, counters,
                           nullptr, b, B))
        return rc;
    if (w_mode != 0 && w_mode != 1) return fail(G6R_EINVAL, "w_mode must be 0 or 1");
    if (!spatial_scale || !grad_image) return fail(G6R_EINVAL, "NULL argument");
    if (scene->n > 0 && (!mu_p || !mu_d || !cov_raw || !sh || !g_mu_p || !g_mu_d || !g_cov_raw ||
                         !g_sh || !g_opacity_raw))
        return fail(G6R_EINVAL, "NULL scene or gradient array");
    char *base = static_cast<char *>(workspace);
    const int rc = launch_backward(
        b.vp[0], *scene, b.ws[0], counters, reinterpret_cast<double *>(base + B.final_t),
        reinterpret_cast<int32_t *>(base + B.last), grad_image,
        reinterpret_cast<int64_t *>(base + B.gids), reinterpret_cast<uint8_t *>(base + B.drawn),
        reinterpret_cast<double *>(base + B.egrad),
        reinterpret_cast<double *>(base + B.gsplat), mu_p, mu_d, cov_raw, sh, spatial_scale,
        directional_scale, w_mode, g_mu_p, g_mu_d, g_cov_raw, g_sh, g_opacity_raw,
        (cudaStream_t)stream);
    if (rc) return rc == G6R_EINVAL ? fail(rc, "backward: bad view") : cuda_check("backward");
    return G6R_OK;
}

int g6r_render_backward(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
                        const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                        int64_t entry_capacity, const double *mu_p, const double *mu_d,
                        const double *cov_raw, const double *sh, const double *spatial_scale,
                        double directional_scale, int32_t w_mode, const double *grad_image,
                        double *g_mu_p, double *g_mu_d, double *g_cov_raw, double *g_sh,
                        double *g_opacity_raw, int64_t *counters, double *image_out,
                        g6r_stream_t stream) {
    if (int rc = g6r_backward_forward(scene, group_mask, cam, cfg, workspace, workspace_bytes,
                                      entry_capacity, counters, image_out, stream))
        return rc;
    return g6r_backward_apply(scene, cam, cfg, workspace, workspace_bytes, entry_capacity, mu_p,
                              mu_d, cov_raw, sh, spatial_scale, directional_scale, w_mode,
                              grad_image, g_mu_p, g_mu_d, g_cov_raw, g_sh, g_opacity_raw, counters,
                              stream);
}

int g6r_decode_records(int64_t n, const void *records, double *mu_p, double *mu_d,
                       double *cov_raw, double *sh, double *opacity_raw, uint8_t *labels,
                       int32_t *bad, g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "decode: n must be >= 0");
    if (n && (!records || !mu_p || !mu_d || !cov_raw || !sh || !opacity_raw || !labels || !bad))
        return fail(G6R_EINVAL, "decode: null pointer");
    if (reinterpret_cast<uintptr_t>(records) & 7) return fail(G6R_EINVAL, "decode: records must be 8-byte aligned");
    if (launch_decode_records(n, records, mu_p, mu_d, cov_raw, sh, opacity_raw, labels, bad,
                              (cudaStream_t)stream))
        return cuda_check("decode_records");
    return G6R_OK;
}

size_t g6r_compact_workspace_bytes(int64_t n) { return compact_workspace_bytes(n); }

int g6r_decode_param_volume_count(const int32_t *dims, const uint8_t *labels_half, void *workspace,
                                  size_t workspace_bytes, int64_t *count, g6r_stream_t stream) {
    if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
        return fail(G6R_EINVAL, "psi decode: dims must be positive");
    const int64_t V = (int64_t)dims[0] * dims[1] * dims[2];
    if (!labels_half || !count || !workspace) return fail(G6R_EINVAL, "psi decode: null pointer");
    if (workspace_bytes < compact_workspace_bytes(V))
        return fail(G6R_EINVAL, "psi decode: workspace too small");
    if (launch_decode_count(V, labels_half, workspace, count, (cudaStream_t)stream))
        return cuda_check("decode_count");
    return G6R_OK;
}

int g6r_decode_param_volume(const int32_t *dims, const void *psi, int32_t psi_f32,
                            const double *base_rgba, const uint8_t *labels_half,
                            const double *spacing, const double *origin, const double *direction,
                            void *workspace, size_t workspace_bytes, double *mu_p, double *mu_d,
                            double *cov_raw, double *sh, double *opacity_raw, uint8_t *labels,
                            g6r_stream_t stream) {
    if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
        return fail(G6R_EINVAL, "psi decode: dims must be positive");
    if (!psi || !base_rgba || !labels_half || !spacing || !origin || !direction || !workspace ||
        !mu_p || !mu_d || !cov_raw || !sh || !opacity_raw || !labels)
        return fail(G6R_EINVAL, "psi decode: null pointer");
    DecodeArgsHost h{};
    h.V = (int64_t)dims[0] * dims[1] * dims[2];
    if (workspace_bytes < compact_workspace_bytes(h.V))
        return fail(G6R_EINVAL, "psi decode: workspace too small");
    h.psi = psi;
    h.psi_f32 = psi_f32 != 0;
    h.base = base_rgba;
    h.lab = labels_half;
    h.dh = dims[1];
    h.dw = dims[2];
    for (int k = 0; k < 3; ++k) {
        h.spacing[k] = spacing[k];
        h.origin[k] = origin[k];
    }
    for (int k = 0; k < 9; ++k) h.dir[k] = direction[k];
    h.mu_p = mu_p;
    h.mu_d = mu_d;
    h.cov_raw = cov_raw;
    h.sh = sh;
    h.opacity_raw = opacity_raw;
    h.labels = labels;
    if (launch_decode_emit(h, workspace, (cudaStream_t)stream)) return cuda_check("decode_emit");
    return G6R_OK;
}

int g6r_filter_rows(int64_t n, const uint8_t *labels, uint32_t group_mask, const double *mu_p,
                    const double *mu_d, const double *cov_raw, const double *sh,
                    const double *opacity_raw, void *workspace, size_t workspace_bytes,
                    double *out_mu_p, double *out_mu_d, double *out_cov_raw, double *out_sh,
                    double *out_opacity_raw, uint8_t *out_labels, int64_t *count,
                    g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "filter: n must be >= 0");
    if (!count || !workspace) return fail(G6R_EINVAL, "filter: null pointer");
    if (n && (!labels || !mu_p || !mu_d || !cov_raw || !sh || !opacity_raw || !out_mu_p ||
              !out_mu_d || !out_cov_raw || !out_sh || !out_opacity_raw || !out_labels))
        return fail(G6R_EINVAL, "filter: null pointer");
    if (workspace_bytes < compact_workspace_bytes(n)) return fail(G6R_EINVAL, "filter: workspace too small");
    const double *in[5] = {mu_p, mu_d, cov_raw, sh, opacity_raw};
    double *out[5] = {out_mu_p, out_mu_d, out_cov_raw, out_sh, out_opacity_raw};
    if (launch_filter_rows(n, labels, group_mask, in, out, out_labels, workspace, count,
                           (cudaStream_t)stream))
        return cuda_check("filter_rows");
    return G6R_OK;
}

size_t g6r_loss_workspace_bytes(int32_t width, int32_t height) {
    if (width <= 0 || height <= 0) return 0;
    return loss_workspace_bytes(height, width);
}

int g6r_loss_grad(const double *pred, const double *target, int32_t target_channels,
                  int32_t width, int32_t height, double lambda_l1, double lambda_ssim,
                  int32_t scales, const double *weights, void *workspace, size_t workspace_bytes,
                  double *grad_out, double *parts, g6r_stream_t stream) {
    if (!pred || !target || !grad_out || !parts || !workspace)
        return fail(G6R_EINVAL, "loss: null pointer");
    if (target_channels != 3 && target_channels != 4)
        return fail(G6R_EINVAL, "loss: target must have 3 or 4 channels");
    if (width < 11 || height < 11) return fail(G6R_EINVAL, "loss: images must be >= 11 px per side");
    if (scales < 1 || scales > 5 || !weights) return fail(G6R_EINVAL, "loss: scales must be 1..5");
    if (!std::isfinite(lambda_l1) || !std::isfinite(lambda_ssim) || lambda_l1 < 0.0 ||
        lambda_ssim < 0.0 || (lambda_l1 == 0.0 && lambda_ssim == 0.0))
        return fail(G6R_EINVAL, "loss: weights must be finite and non-negative, one positive");
    for (int j = 0; j < scales; ++j)
        if (!std::isfinite(weights[j])) return fail(G6R_EINVAL, "loss: scale weights must be finite");
    if (workspace_bytes < loss_workspace_bytes(height, width))
        return fail(G6R_EINVAL, "loss: workspace too small");
    if (loss_grad(pred, target, target_channels, height, width, lambda_l1, lambda_ssim, scales,
                  weights, workspace, grad_out, parts, (cudaStream_t)stream))
        return cuda_check("loss_grad");
    return G6R_OK;
}

int g6r_adam_step(int64_t count, double *param, const double *grad, double *m, double *v,
                  double lr, double bias1, double bias2, g6r_stream_t stream) {
    if (count < 0) return fail(G6R_EINVAL, "adam: count must be >= 0");
    if (adam_step(count, param, grad, m, v, lr, bias1, bias2, (cudaStream_t)stream))
        return cuda_check("adam_step");
    return G6R_OK;
}

int g6r_any_nonfinite(int64_t count, const double *x, int32_t *flag, g6r_stream_t stream) {
    if (count < 0) return fail(G6R_EINVAL, "nonfinite: count must be >= 0");
    if (nonfinite(count, x, flag, (cudaStream_t)stream)) return cuda_check("nonfinite");
    return G6R_OK;
}

int g6r_debug_expf(int64_t n, const float *x, float *y, g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "n must be >= 0");
    if (launch_debug_expf(n, x, y, (cudaStream_t)stream)) return cuda_check("debug_expf");
    return G6R_OK;
}

int g6r_debug_exp(int64_t n, const double *x, double *y, g6r_stream_t stream) {
    if (n < 0) return fail(G6R_EINVAL, "n must be >= 0");
    if (launch_debug_exp(n, x, y, (cudaStream_t)stream)) return cuda_check("debug_exp");
    return G6R_OK;
}

int g6r_project(const g6r_scene *scene, uint32_t group_mask, const g6r_camera *cam,
                const g6r_config *cfg, void *workspace, size_t workspace_bytes,
                int64_t *counters, const g6r_splat_out *splats, g6r_stream_t stream) {
    if (!scene || scene->n < 0) return fail(G6R_EINVAL, "scene is NULL");
    if (!counters) return fail(G6R_EINVAL, "counters are required");
    Batch b;
    memset(&b, 0, sizeof b);
    b.nviews = 1;
    if (int rc = make_view(cam, cfg, b.vp[0])) return rc;
    const Layout L = layout(scene->n, (int64_t)b.vp[0].tiles_x * b.vp[0].tiles_y, 0, b.vp[0].precision);
    if (int rc = check_ws(L.total, workspace, workspace_bytes)) return rc;
    b.ws[0] = carve(workspace, L, 0);
    b.out[0].counters = counters;
    cudaStream_t st = (cudaStream_t)stream;
    if (launch_clear(b, L.clear_end, st)) return cuda_check("clear");
    if (launch_project(*scene, group_mask, b, splats, false, st)) return cuda_check("project");
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
    Batch b;
    memset(&b, 0, sizeof b);
    b.nviews = 1;
    ViewParams &vp = b.vp[0];
    vp.iw = width;
    vp.ih = height;
    vp.tile_size = tile_size;
    vp.tiles_x = (width + tile_size - 1) / tile_size;
    vp.tiles_y = (height + tile_size - 1) / tile_size;
    const Layout L = layout(m, (int64_t)vp.tiles_x * vp.tiles_y, entry_capacity, 0);
    if (int rc = check_ws(L.total, workspace, workspace_bytes)) return rc;
    b.ws[0] = carve(workspace, L, entry_capacity);
    b.out[0].counters = counters;
    b.out[0].entry_splat = entry_splat;
    b.out[0].tile_starts = tile_starts;
    cudaStream_t st = (cudaStream_t)stream;
    if (launch_clear(b, L.clear_end, st)) return cuda_check("clear");
    if (launch_duplicate(m, means2d, radii, depths, b, st)) return cuda_check("duplicate");
    if (launch_sort(b, m, st)) return cuda_check("sort");
    if (launch_ranges(b, m, st)) return cuda_check("ranges");
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
    if (int rc = check_ws(L.total, workspace, workspace_bytes)) return rc;
    Batch b;
    memset(&b, 0, sizeof b);
    b.nviews = 1;
    ViewParams &vp = b.vp[0];
    vp.iw = width;
    vp.ih = height;
    vp.tile_size = tile_size;
    vp.tiles_x = tiles_x;
    vp.tiles_y = tiles_y;
    vp.precision = precision;
    b.ws[0] = carve(workspace, L, 0);
    b.ws[0].vals[0] = const_cast<unsigned *>(reinterpret_cast<const unsigned *>(entry_splat));
    b.ws[0].tile_starts = const_cast<int64_t *>(tile_starts);
    b.out[0].image = image;
    b.out[0].final_t = final_t;
    b.out[0].last_contrib = last_contrib;
    cudaStream_t st = (cudaStream_t)stream;
    if (launch_pack_payload(m, precision, means2d, conics, colors, alphas, b.ws[0].payload, st))
        return cuda_check("pack_payload");
    if (launch_composite(b, false, st)) return cuda_check("composite");
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
