// g6r_sort.cu -- on-device stable LSD radix sort of the tile entries and
// per-tile range extraction.
//
// Replaces raster.py:376-379: np.argsort(key, kind="stable") over the 64-bit
// keys (tile << 32 | f32 depth bits) and tile_starts = cumsum(bincount(tile)).
// Stability reproduces the reference tie rule (equal keys keep splat order,
// raster.py:22-24), so the output is bit-identical to the reference.
//
// Design: one histogram launch computes every pass's digit counts at once
// (LSD digit counts do not depend on the order), then one "onesweep" launch
// per 8-bit digit: each CTA ranks a 4096-key tile with warp match-any, gets
// its global digit offsets by decoupled look-back over earlier tiles, and
// scatters.  Tiles are claimed through an atomic ticket so a CTA only ever
// waits on tiles already owned by running CTAs.  E is read on the device;
// grids are sized from the capacity and idle CTAs exit, so there is no host
// round trip between projection and compositing.
#include <algorithm>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

constexpr unsigned kAgg = 1u << 30, kInc = 2u << 30, kCntMask = (1u << 30) - 1;

int sort_passes(int tiles) {
    int tb = 0;
    while ((1ll << tb) < (long long)tiles) ++tb;
    return (32 + tb + 7) / 8;
}

__device__ __forceinline__ bool entries_valid(const int64_t *counters, int64_t cap, int64_t &e) {
    e = counters[G6R_CNT_ENTRIES];
    return !counters[G6R_CNT_OVERFLOW] && e <= cap;
}

__global__ void __launch_bounds__(kBlock)
k_sort_hist(const unsigned long long *__restrict__ keys, const int64_t *counters, int64_t cap,
            int passes, unsigned *__restrict__ hist, unsigned *__restrict__ status,
            int64_t tiles_cap) {
    __shared__ unsigned h[kMaxPasses][256];
    int64_t e;
    if (!entries_valid(counters, cap, e)) return;
    const int64_t ntiles = ceil_div(e, kSortTile);
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (int64_t k = gtid; k < ntiles * 256; k += gsz) status[p * tiles_cap * 256 + k] = 0u;
    for (int k = threadIdx.x; k < kMaxPasses * 256; k += blockDim.x) (&h[0][0])[k] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < e; base += gsz) {
        const int64_t idx = base + threadIdx.x;
        const bool valid = idx < e;
        const unsigned long long key = valid ? keys[idx] : 0ull;
        for (int p = 0; p < passes; ++p) {
            const unsigned d = valid ? (unsigned)((key >> (8 * p)) & 255ull) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256u && lane == __ffs(peers) - 1) atomicAdd(&h[p][d], (unsigned)__popc(peers));
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < passes * 256; k += blockDim.x) {
        const unsigned v = (&h[0][0])[k];
        if (v) atomicAdd(&hist[k], v);
    }
}

__global__ void __launch_bounds__(kBlock)
k_onesweep(const unsigned long long *__restrict__ kin, const unsigned *__restrict__ vin,
           unsigned long long *__restrict__ kout, unsigned *__restrict__ vout,
           const int64_t *counters, int64_t cap, int shift, const unsigned *__restrict__ hist_p,
           unsigned *status_p, unsigned long long *ticket) {
    __shared__ unsigned s_goff[256];
    __shared__ unsigned s_wh[kBlock / 32][256];
    __shared__ unsigned s_base[256];
    __shared__ unsigned s_scan[kBlock / 32];
    __shared__ int64_t s_tile;
    int64_t e;
    if (!entries_valid(counters, cap, e)) return;
    const int64_t ntiles = ceil_div(e, kSortTile);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {   // global exclusive digit offsets of this pass (block scan of 256 counts)
        const unsigned c = hist_p[tid];
        const unsigned inc = warp_inclusive_scan(c);
        if (lane == 31) s_scan[warp] = inc;
        __syncthreads();
        unsigned pre = 0;
        for (int w = 0; w < warp; ++w) pre += s_scan[w];
        s_goff[tid] = pre + inc - c;
    }
    const unsigned lanemask_lt = (1u << lane) - 1u;
    while (true) {
        if (tid == 0) s_tile = (int64_t)atomicAdd(ticket, 1ull);
#pragma unroll
        for (int w = 0; w < kBlock / 32; ++w) s_wh[w][tid] = 0u;
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= ntiles) break;
        const int64_t base = tile * kSortTile + (int64_t)warp * (32 * kSortItems);
        unsigned long long key[kSortItems];
        unsigned val[kSortItems];
        unsigned rank[kSortItems];
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * 32 + lane;
            const bool valid = idx < e;
            key[k] = valid ? kin[idx] : ~0ull;
            val[k] = valid ? vin[idx] : 0u;
            rank[k] = valid ? 0u : 0xffffffffu;
        }
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const unsigned d = rank[k] == 0xffffffffu ? 256u : (unsigned)((key[k] >> shift) & 255ull);
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const int leader = __ffs(peers) - 1;
            unsigned old = 0;
            if (d < 256u && lane == leader) {
                old = s_wh[warp][d];
                s_wh[warp][d] = old + (unsigned)__popc(peers);
            }
            old = __shfl_sync(0xffffffffu, old, leader);
            if (d < 256u) rank[k] = old + (unsigned)__popc(peers & lanemask_lt);
            __syncwarp();
        }
        __syncthreads();
        // per digit: exclusive prefix over warps, CTA total, look-back
        unsigned run = 0;
#pragma unroll
        for (int w = 0; w < kBlock / 32; ++w) {
            const unsigned c = s_wh[w][tid];
            s_wh[w][tid] = run;
            run += c;
        }
        unsigned *my = status_p + tile * 256 + tid;
        unsigned excl = 0;
        if (tile == 0) {
            st_volatile_u32(my, kInc | run);
        } else {
            st_volatile_u32(my, kAgg | run);
            int64_t j = tile - 1;
            while (true) {
                const unsigned w = ld_volatile_u32(status_p + j * 256 + tid);
                const unsigned fl = w & ~kCntMask;
                if (!fl) continue;
                excl += w & kCntMask;
                if (fl == kInc) break;
                --j;
            }
            st_volatile_u32(my, kInc | (excl + run));
        }
        s_base[tid] = s_goff[tid] + excl;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            if (rank[k] == 0xffffffffu) continue;
            const unsigned d = (unsigned)((key[k] >> shift) & 255ull);
            const unsigned pos = s_base[d] + s_wh[warp][d] + rank[k];
            kout[pos] = key[k];
            vout[pos] = val[k];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kBlock)
k_ranges(const unsigned long long *__restrict__ keys, const unsigned *__restrict__ vals,
         const int64_t *counters, int64_t cap, int64_t n_tiles, int64_t *__restrict__ starts,
         int64_t *__restrict__ starts2, int32_t *__restrict__ entry_out) {
    int64_t e;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
    if (!entries_valid(counters, cap, e)) {   // overflow: empty runs everywhere
        for (int64_t t = gtid; t <= n_tiles; t += gsz) {
            starts[t] = 0;
            if (starts2) starts2[t] = 0;
        }
        return;
    }
    for (int64_t i = gtid; i <= e; i += gsz) {
        const int64_t ti = i < e ? (int64_t)(keys[i] >> 32) : n_tiles;
        const int64_t tp = i > 0 ? (int64_t)(keys[i - 1] >> 32) : -1;
        for (int64_t t = tp + 1; t <= ti; ++t) {
            starts[t] = i;
            if (starts2) starts2[t] = i;
        }
        if (i < e && entry_out) entry_out[i] = (int32_t)vals[i];
    }
}

static int num_sms() {
    static int cached = 0;
    if (!cached) {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
        cached = v;
    }
    return cached;
}

int launch_sort(const ViewParams &vp, const Workspace &ws, const int64_t *counters, int *final_buf,
                cudaStream_t st) {
    const int64_t n_tiles = (int64_t)vp.tiles_x * vp.tiles_y;
    const int passes = sort_passes((int)n_tiles);
    const int64_t cap = ws.entry_capacity;
    const int sms = num_sms();
    const unsigned hist_grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, kBlock), sms * 4));
    k_sort_hist<<<hist_grid, kBlock, 0, st>>>(ws.keys[0], counters, cap, passes, ws.hist,
                                              ws.sort_status, ws.sort_tiles_cap);
    int src = 0;
    const unsigned sweep_grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ws.sort_tiles_cap, sms * 3));
    for (int p = 0; p < passes; ++p) {
        k_onesweep<<<sweep_grid, kBlock, 0, st>>>(
            ws.keys[src], ws.vals[src], ws.keys[1 - src], ws.vals[1 - src], counters, cap, 8 * p,
            ws.hist + p * 256, ws.sort_status + (int64_t)p * ws.sort_tiles_cap * 256,
            reinterpret_cast<unsigned long long *>(&ws.internal[kTicketSortBase + p]));
        src = 1 - src;
    }
    *final_buf = src;
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_ranges(const ViewParams &vp, const Workspace &ws, const int64_t *counters, int buf,
                  int64_t *tile_starts_out, int32_t *entry_splat_out, cudaStream_t st) {
    const int64_t n_tiles = (int64_t)vp.tiles_x * vp.tiles_y;
    const int64_t cap = ws.entry_capacity;
    const unsigned rgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap + 1, kBlock), num_sms() * 4));
    k_ranges<<<rgrid, kBlock, 0, st>>>(ws.keys[buf], ws.vals[buf], counters, cap, n_tiles,
                                       ws.tile_starts, tile_starts_out, entry_splat_out);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
