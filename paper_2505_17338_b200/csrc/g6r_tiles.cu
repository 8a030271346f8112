// g6r_tiles.cu -- order-preserving expansion of depth-sorted splats into
// per-tile runs (the splat-level half of the hot-path sort).
//
// The reference orders every tile's run by (f32 depth bits, then entry order),
// raster.py:366-379.  Entry order follows the splat index and equal depths keep
// it, so the run of tile t is exactly "the drawn splats whose rect covers t, in
// (depth, row) order".  The hot path therefore sorts the n splat rows by depth
// once (g6r_sort.cu, splat mode: n keys instead of E entries, 8-byte items) and
// expands them here without a second sort:
//   k_chunk_count    per chunk of chunk_splats(T) sorted splats: tile histogram
//   k_chunk_colscan  per tile: exclusive prefix over chunks, tile totals
//   k_tile_scan      tile_starts = exclusive scan of the totals (+ overflow)
//   k_chunk_scatter  per chunk, in rounds of 256 splats: the round's entries
//                    are expanded in order into a shared window, each warp
//                    ranks a contiguous slice of the window with match-any on
//                    the tile id and 16-bit per-warp counters, the counters are
//                    prefixed over warps, and every entry's splat row is
//                    written to tile_start + chunk prefix + running count +
//                    warp prefix + rank.
// Every step is deterministic and keeps the sorted order, so runs, tile starts
// and images are bit-identical to the entry sort's.
#include <algorithm>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

constexpr int kScatterWarps = 8;

struct PartCtx {
    int64_t m;             // drawn splats (the first m sorted items)
    int64_t chunks;
    int chunk;             // sorted splats per chunk
    int tiles, tiles_x;
    const unsigned long long *items;   // depth-sorted (depth code << vbits | row)
};

__device__ __forceinline__ bool part_ctx(const Batch &b, int v, PartCtx &c) {
    const int64_t *cnt = b.out[v].counters;
    const Workspace &ws = b.ws[v];
    if (cnt[G6R_CNT_OVERFLOW] || cnt[G6R_CNT_ENTRIES] > ws.entry_capacity) return false;
    c.m = cnt[G6R_CNT_DRAWN];
    c.tiles_x = b.vp[v].tiles_x;
    c.tiles = b.vp[v].tiles_x * b.vp[v].tiles_y;
    c.chunk = chunk_splats(c.tiles);
    c.chunks = ceil_div(c.m, c.chunk);
    c.items = ws.keys[ws.internal[kSortPasses] & 1];
    return true;
}

__device__ __forceinline__ void unpack_rect(uint2 r, int &x0, int &y0, int &wx, int &hy) {
    x0 = (int)(r.x & 0xffffu);
    y0 = (int)(r.x >> 16);
    wx = (int)(r.y & 0xffffu);
    hy = (int)(r.y >> 16);
}

__global__ void __launch_bounds__(kBlock)
k_chunk_count(const __grid_constant__ Batch b, unsigned long long vmask) {
    extern __shared__ unsigned s_hist[];
    const int v = blockIdx.y;
    PartCtx c;
    if (!part_ctx(b, v, c) || blockIdx.x >= c.chunks) return;
    const Workspace &ws = b.ws[v];
    for (int t = threadIdx.x; t < c.tiles; t += blockDim.x) s_hist[t] = 0u;
    __syncthreads();
    const int64_t s0 = (int64_t)blockIdx.x * c.chunk;
    const int64_t s1 = s0 + c.chunk < c.m ? s0 + c.chunk : c.m;
    for (int64_t sp = s0 + threadIdx.x; sp < s1; sp += blockDim.x) {
        const unsigned row = (unsigned)(c.items[sp] & vmask);
        int x0, y0, wx, hy;
        unpack_rect(ws.rect[row], x0, y0, wx, hy);
        for (int yy = 0; yy < hy; ++yy)
            for (int xx = 0; xx < wx; ++xx) atomicAdd(&s_hist[(y0 + yy) * c.tiles_x + x0 + xx], 1u);
    }
    __syncthreads();
    unsigned *row_out = ws.chunk_hist + (int64_t)blockIdx.x * c.tiles;
    for (int t = threadIdx.x; t < c.tiles; t += blockDim.x) row_out[t] = s_hist[t];
}

// Exclusive prefix of every tile column over the chunks, and the tile totals.
// CTA x owns 32 tiles (lane = tile); its 8 warps each sum a contiguous range of
// chunks, the range sums are scanned in shared memory, then each warp rewrites
// its range.
__global__ void __launch_bounds__(kBlock) k_chunk_colscan(const __grid_constant__ Batch b) {
    __shared__ unsigned s_sum[kBlock / 32][32];
    const int v = blockIdx.y;
    PartCtx c;
    if (!part_ctx(b, v, c)) return;
    const Workspace &ws = b.ws[v];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kBlock / 32;
    const int t = blockIdx.x * 32 + lane;
    const bool ok = t < c.tiles;
    const int64_t per = ceil_div(c.chunks, nw);
    const int64_t a = warp * per, e = a + per < c.chunks ? a + per : c.chunks;
    constexpr int U = 8;
    unsigned sum = 0;
    for (int64_t ch = a; ch < e; ch += U) {
        unsigned x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (ok && ch + u < e) ? ws.chunk_hist[(ch + u) * c.tiles + t] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) sum += x[u];
    }
    s_sum[warp][lane] = sum;
    __syncthreads();
    unsigned run = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
        const unsigned x = s_sum[w][lane];
        run += w < warp ? x : 0u;
        total += x;
    }
    for (int64_t ch = a; ch < e; ch += U) {
        unsigned x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (ok && ch + u < e) ? ws.chunk_hist[(ch + u) * c.tiles + t] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (ok && ch + u < e) ws.chunk_hist[(ch + u) * c.tiles + t] = run;
            run += x[u];
        }
    }
    if (ok && warp == 0) ws.tile_total[t] = total;
}

// one CTA per view: tile_starts (T+1) from the totals; empty runs on overflow
__global__ void __launch_bounds__(1024) k_tile_scan(const __grid_constant__ Batch b) {
    __shared__ unsigned long long s_warp[32];
    __shared__ unsigned long long s_carry;
    const int v = blockIdx.y;
    const Workspace &ws = b.ws[v];
    int64_t *starts = ws.tile_starts;
    int64_t *starts2 = b.out[v].tile_starts;
    const int tiles = b.vp[v].tiles_x * b.vp[v].tiles_y;
    PartCtx c;
    if (!part_ctx(b, v, c)) {
        for (int t = threadIdx.x; t <= tiles; t += blockDim.x) {
            starts[t] = 0;
            if (starts2) starts2[t] = 0;
        }
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int t0 = 0; t0 < tiles; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const unsigned long long x = t < tiles ? ws.tile_total[t] : 0ull;
        const unsigned long long inc = warp_inclusive_scan(x);
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long w = s_warp[lane];
            s_warp[lane] = warp_inclusive_scan(w) - w;
        }
        __syncthreads();
        const unsigned long long excl = s_carry + s_warp[warp] + inc - x;
        if (t < tiles) {
            starts[t] = (int64_t)excl;
            if (starts2) starts2[t] = (int64_t)excl;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = excl + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        starts[tiles] = (int64_t)s_carry;
        if (starts2) starts2[tiles] = (int64_t)s_carry;
    }
}

constexpr int kPerThread = 4;                 // sorted splats per thread per round
constexpr int kRound = kBlock * kPerThread;   // 1024 splats per round
constexpr int kWindow = 4096;                 // expanded entries ranked at a time
constexpr int kWinPerWarp = kWindow / kScatterWarps;   // 512: 16 groups of 32
constexpr int kGroups = kWinPerWarp / 32;
constexpr size_t kScatterStatic = (size_t)kWindow * (2 * sizeof(unsigned) + sizeof(unsigned short));

__global__ void __launch_bounds__(kBlock)
k_chunk_scatter(const __grid_constant__ Batch b, unsigned long long vmask) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    __shared__ unsigned s_wsum[kScatterWarps];
    const int v = blockIdx.y;
    PartCtx c;
    if (!part_ctx(b, v, c) || blockIdx.x >= c.chunks) return;
    const Workspace &ws = b.ws[v];
    // dynamic shared memory: window (tile, row, rank), then per-tile state
    unsigned *s_ewin = reinterpret_cast<unsigned *>(s_raw);                    // [kWindow]
    unsigned *s_rwin = s_ewin + kWindow;                                       // [kWindow]
    unsigned short *s_rank = reinterpret_cast<unsigned short *>(s_rwin + kWindow);   // [kWindow]
    unsigned *s_base = reinterpret_cast<unsigned *>(s_rank + kWindow);         // [T]
    unsigned short *s_cnt = reinterpret_cast<unsigned short *>(s_base + c.tiles);   // [warps][T]
    unsigned short *s_tot = s_cnt + kScatterWarps * c.tiles;                        // [T]
    const unsigned *chunk_off = ws.chunk_hist + (int64_t)blockIdx.x * c.tiles;
    for (int t = threadIdx.x; t < c.tiles; t += blockDim.x)
        s_base[t] = (unsigned)ws.tile_starts[t] + chunk_off[t];
    for (int k = threadIdx.x; k < kScatterWarps * c.tiles; k += blockDim.x) s_cnt[k] = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    unsigned *vals = ws.vals[0];
    const int64_t c0 = (int64_t)blockIdx.x * c.chunk;
    const int64_t c1 = c0 + c.chunk < c.m ? c0 + c.chunk : c.m;
    for (int64_t r0 = c0; r0 < c1; r0 += kRound) {
        // this thread's kPerThread consecutive splats of the round
        unsigned row[kPerThread];
        uint2 rc[kPerThread];
        int cnt_all = 0;
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            const int64_t sp = r0 + threadIdx.x * kPerThread + q;
            row[q] = sp < c1 ? (unsigned)(c.items[sp] & vmask) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            const int64_t sp = r0 + threadIdx.x * kPerThread + q;
            rc[q] = sp < c1 ? ws.rect[row[q]] : make_uint2(0u, 0u);
            cnt_all += (int)((rc[q].y & 0xffffu) * (rc[q].y >> 16));
        }
        const int inc = warp_inclusive_scan(cnt_all);
        __syncthreads();   // previous round's window and s_wsum are free
        if (lane == 31) s_wsum[warp] = (unsigned)inc;
        __syncthreads();
        int pre = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kScatterWarps; ++w) {
            const int x = (int)s_wsum[w];
            pre += w < warp ? x : 0;
            total += x;
        }
        const int off0 = pre + inc - cnt_all;   // first entry of this thread's splats
        for (int w0 = 0; w0 < total; w0 += kWindow) {
            const int wn = total - w0 < kWindow ? total - w0 : kWindow;
            // expand this thread's entries inside [w0, w0 + wn), in order
            int off = off0;
#pragma unroll
            for (int q = 0; q < kPerThread; ++q) {
                int x0, y0, wx, hy;
                unpack_rect(rc[q], x0, y0, wx, hy);
                const int cnt = wx * hy;
                const int k_lo = w0 > off ? w0 - off : 0;
                const int k_hi = off + cnt < w0 + wn ? cnt : w0 + wn - off;
                if (k_lo < k_hi) {   // row-major walk of the rect from entry k_lo
                    int qy = k_lo / wx, qx = k_lo - qy * wx;
                    unsigned t = (unsigned)((y0 + qy) * c.tiles_x + x0 + qx);
                    for (int k = k_lo; k < k_hi; ++k) {
                        s_ewin[off + k - w0] = t;
                        s_rwin[off + k - w0] = row[q];
                        if (++qx == wx) {
                            qx = 0;
                            t += (unsigned)(c.tiles_x - wx + 1);
                        } else {
                            ++t;
                        }
                    }
                }
                off += cnt;
            }
            __syncthreads();
            // rank: warp w owns window slots [w*512, w*512+512), 32 at a time in order
#pragma unroll 4
            for (int g = 0; g < kGroups; ++g) {
                const int slot = warp * kWinPerWarp + g * 32 + lane;
                const bool valid = slot < wn;
                const unsigned t = valid ? s_ewin[slot] : 0xffffffffu;
                const unsigned peers = __match_any_sync(0xffffffffu, t);
                const int leader = __ffs(peers) - 1;
                unsigned old = 0;
                if (valid && lane == leader) {
                    old = s_cnt[warp * c.tiles + t];
                    s_cnt[warp * c.tiles + t] = (unsigned short)(old + (unsigned)__popc(peers));
                }
                old = __shfl_sync(0xffffffffu, old, leader);
                if (valid) s_rank[slot] = (unsigned short)(old + (unsigned)__popc(peers & lanemask_lt));
                __syncwarp();
            }
            __syncthreads();
            // per tile: the warp counts become exclusive offsets (warps in order)
            for (int t = threadIdx.x; t < c.tiles; t += blockDim.x) {
                unsigned run = 0;
#pragma unroll
                for (int w = 0; w < kScatterWarps; ++w) {
                    const unsigned x = s_cnt[w * c.tiles + t];
                    s_cnt[w * c.tiles + t] = (unsigned short)run;
                    run += x;
                }
                s_tot[t] = (unsigned short)run;
            }
            __syncthreads();
            // scatter: tile base + warp offset + rank
            for (int slot = threadIdx.x; slot < wn; slot += blockDim.x) {
                const unsigned t = s_ewin[slot];
                vals[s_base[t] + s_cnt[(slot / kWinPerWarp) * c.tiles + t] + s_rank[slot]] = s_rwin[slot];
            }
            __syncthreads();
            // advance the bases by this window's counts and clear the counters
            for (int t = threadIdx.x; t < c.tiles; t += blockDim.x) {
                s_base[t] += s_tot[t];
#pragma unroll
                for (int w = 0; w < kScatterWarps; ++w) s_cnt[w * c.tiles + t] = 0;
            }
            __syncthreads();
        }
    }
}

int launch_tile_partition(const Batch &b, int64_t n, int vbits, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    const int tiles = b.vp[0].tiles_x * b.vp[0].tiles_y;
    const int64_t chunks = ceil_div(n > 0 ? n : 1, chunk_splats(tiles));
    const unsigned long long vmask = (1ull << vbits) - 1ull;
    const size_t count_smem = (size_t)tiles * sizeof(unsigned);
    const size_t scatter_smem =
        kScatterStatic + (size_t)tiles * (sizeof(unsigned) + (kScatterWarps + 1) * sizeof(unsigned short));
    static bool attrs = false;
    if (!attrs) {
        cudaFuncSetAttribute(k_chunk_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kMaxSplatSortTiles * sizeof(unsigned)));
        cudaFuncSetAttribute(k_chunk_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kScatterStatic + kMaxSplatSortTiles * (sizeof(unsigned) + (kScatterWarps + 1) * sizeof(unsigned short))));
        attrs = true;
    }
    const dim3 cgrid((unsigned)chunks, (unsigned)b.nviews);
    k_chunk_count<<<cgrid, kBlock, count_smem, st>>>(b, vmask);
    trace_mark("chunk_count", st);
    k_chunk_colscan<<<dim3((unsigned)ceil_div(tiles, 32), b.nviews), kBlock, 0, st>>>(b);
    trace_mark("chunk_colscan", st);
    k_tile_scan<<<dim3(1, b.nviews), 1024, 0, st>>>(b);
    trace_mark("tile_scan", st);
    k_chunk_scatter<<<cgrid, kBlock, scatter_smem, st>>>(b, vmask);
    trace_mark("chunk_scatter", st);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
