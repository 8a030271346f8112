// g6r_sort.cu -- on-device stable LSD radix sort of the tile entries and
// per-tile range extraction, for a batch of views per launch.
//
// Replaces raster.py:376-379: np.argsort(key, kind="stable") over the 64-bit
// keys (tile << 32 | f32 depth bits) and tile_starts = cumsum(bincount(tile)).
// Stability reproduces the reference tie rule (equal keys keep splat order,
// raster.py:22-24), so the output is bit-identical to the reference.
//
// Key compression: depths are positive, so their f32 bit patterns order
// monotonically; the projection records the view's min/max depth bits and the
// sort ranks the order-preserving key' = tile << dbits | (depth_bits - dmin)
// with dbits = bits(dmax - dmin).  At 512^2 with a 1M-Gaussian orbit view that
// is ~10 + 24 bits: 4 passes of 9-bit digits instead of 6 passes of 8 bits.
// The stored keys stay the original 64-bit keys (ranges read the tile from
// them); digits are computed on the fly.  The pass count is decided on the
// device per view; surplus work exits at once and consumers read which
// ping-pong buffer holds the result (sorted_buffer()).
//
// Each pass is ONE "onesweep" kernel (grid y = view): a CTA claims the next
// 2048-key tile of its view through an atomic ticket, ranks the tile's keys
// (stable: warp-striped items, warps in order), publishes the tile's digit
// counts, and finds its global digit offsets by decoupled look-back over the
// earlier tiles' status words (2-bit flag | 30-bit count in one 32-bit word,
// so a single store publishes both and no fence is needed).  The look-back
// reads the immediate predecessor, then 4 per round trip.  One histogram
// launch before the passes computes every pass's digit totals (LSD digit
// counts do not depend on the order) and zeroes the status words.  With a
// batch of views per launch the views' look-back chains run side by side.
// Pass 0 packs key and value into one u64 (tile | depth code | value) when
// they fit, so later passes move 8 bytes per item.
//
// Two item sets use these kernels:
//   * entries (launch_sort): the E (tile, depth) keys of the entry path, then
//     k_ranges;
//   * splats (launch_splat_sort, the hot path): the n scene rows keyed by
//     depth alone -- rows not drawn carry an all-ones key that compresses to
//     one extra code and sorts last -- then the tile partition (g6r_tiles.cu).
#include <algorithm>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

constexpr int kWarps = kBlock / 32;
constexpr int kDigitsPerThread = kBins / kBlock;   // 2

int tile_bits(int64_t tiles) {
    int tb = 0;
    while ((1ll << tb) < tiles) ++tb;
    return tb;
}

int sort_passes(int tiles) {   // upper bound (full 32 depth bits)
    return (32 + tile_bits(tiles) + kRadixBits - 1) / kRadixBits;
}

__device__ __forceinline__ bool entries_valid(const int64_t *counters, int64_t cap, int64_t &e) {
    e = counters[G6R_CNT_ENTRIES];
    return !counters[G6R_CNT_OVERFLOW] && e <= cap;
}

// (dmin, dbits, passes) of a view from the projection's depth-bit extrema.
// With `sentinel` (splat sort) one more code, span + 1, is reserved for rows
// that were not drawn (key all-ones), so they sort after every drawn splat.
// Digit width: the fewest passes of at most kRadixBits bits, then the
// narrowest digit that still covers the key in that many passes (a 23-bit key
// runs as 3 x 8 bits, not 3 x 9): fewer bins make every tile's digit prefix,
// status publication and look-back cheaper (1 digit per thread instead of 2).
__device__ __forceinline__ void view_key_shape(const long long *internal, int tbits, bool sentinel,
                                               unsigned &dmin, unsigned &dtop, int &dbits,
                                               int &passes, int &rbits) {
    const unsigned lo = ~(unsigned)internal[kDepthMinInv];
    const unsigned hi = (unsigned)internal[kDepthMax];
    const unsigned span = hi >= lo ? hi - lo : 0u;
    dmin = hi >= lo ? lo : 0u;
    dtop = span + (sentinel ? 1u : 0u);   // largest compressed depth code
    dbits = dtop ? 32 - __clz(dtop) : 0;
    const int total = tbits + dbits;
    passes = (total + kRadixBits - 1) / kRadixBits;
    rbits = passes ? (total + passes - 1) / passes : kRadixBits;
}

__device__ __forceinline__ unsigned depth_code(unsigned long long key, unsigned dmin, unsigned dtop) {
    const unsigned d = (unsigned)key - dmin;
    return d < dtop ? d : dtop;   // clamps the not-drawn sentinel (and only it)
}

__device__ __forceinline__ unsigned digit_of(unsigned long long key, unsigned dmin, unsigned dtop,
                                             int dbits, int shift, unsigned mask) {
    const unsigned long long k2 =
        ((key >> 32) << dbits) | (unsigned long long)depth_code(key, dmin, dtop);
    return (unsigned)(k2 >> shift) & mask;
}

// Common prologue: this view's entry count, key shape, and whether `pass` runs.
// Packed mode (tile + depth + value bits fit 64): pass 0 folds each entry into
// one u64 `tile << (dbits+vbits) | (depth - dmin) << vbits | value`, so later
// passes move 8 bytes per entry instead of a 12-byte key/value pair.
// Splat mode (splat_n > 0): the items are the scene's n rows (key = f32 depth
// bits or the not-drawn sentinel, value = row), sorted by depth alone.
struct PassCtx {
    int64_t e, ntiles;
    unsigned dmin, dtop;
    int dbits, passes, vbits, rbits;   // rbits: digit width of this view's passes
    unsigned nbins;                    // 1 << rbits (<= kBins)
    bool packed, splat;
};

__device__ __forceinline__ bool pass_ctx(const Batch &b, int v, int tbits, int vbits, int pass,
                                         PassCtx &c, int64_t splat_n = 0) {
    if (!entries_valid(b.out[v].counters, b.ws[v].entry_capacity, c.e)) return false;
    c.splat = splat_n > 0;
    if (c.splat) {
        c.e = splat_n;
        tbits = 0;
    }
    view_key_shape(b.ws[v].internal, tbits, c.splat, c.dmin, c.dtop, c.dbits, c.passes, c.rbits);
    c.nbins = 1u << c.rbits;
    c.ntiles = ceil_div(c.e, kSortTile);
    c.vbits = vbits;
    c.packed = tbits + c.dbits + vbits <= 64;
    return pass < c.passes;
}

__device__ __forceinline__ unsigned long long pack_entry(unsigned long long key, unsigned val,
                                                         const PassCtx &c) {
    return ((key >> 32) << (c.dbits + c.vbits)) |
           ((unsigned long long)depth_code(key, c.dmin, c.dtop) << c.vbits) | (unsigned long long)val;
}

__device__ __forceinline__ int pass_src(int pass) { return pass & 1; }

// Lanes of the warp holding the same (rbits+1)-bit value (digit, or the
// nbins "invalid" code): one ballot per bit instead of MATCH.ANY.
__device__ __forceinline__ unsigned match_digit(unsigned d, int rbits) {
    unsigned peers = 0xffffffffu;
    for (int bit = 0; bit <= rbits; ++bit) {
        const bool on = (d >> bit) & 1u;
        const unsigned b = __ballot_sync(0xffffffffu, on);
        peers &= on ? b : ~b;
    }
    return peers;
}

constexpr unsigned kAgg = 1u << 30, kInc = 2u << 30, kCntMask = (1u << 30) - 1;
constexpr int kProbe = 4;   // look-back predecessors read per round trip

// Digit totals of every pass in one read of the keys; zero the status words.
// Each warp counts into its own shared histogram with plain shared atomics.
constexpr int kHistWarps = 4;   // warp histograms per CTA (warps 2w, 2w+1 share one)
__global__ void __launch_bounds__(kBlock)
k_sort_hist(const __grid_constant__ Batch b, int tbits, int vbits, int64_t splat_n) {
    __shared__ unsigned h[kHistWarps][4][kBins];   // up to 4 passes counted in smem
    const int v = blockIdx.y;
    PassCtx c;
    const bool run = pass_ctx(b, v, tbits, vbits, 0, c, splat_n);
    const Workspace &ws = b.ws[v];
    if (splat_n > 0 && blockIdx.x == 0 && threadIdx.x == 0 &&
        b.out[v].counters[G6R_CNT_ENTRIES] > ws.entry_capacity)
        b.out[v].counters[G6R_CNT_OVERFLOW] = 1;   // the entries will not fit: skip the view
    if (blockIdx.x == 0 && threadIdx.x == 0 && c.e <= ws.entry_capacity) {
        ws.internal[kSortPasses] = run ? c.passes : 0;
        ws.internal[kValsBuffer] = (run && !c.packed) ? (c.passes & 1) : 0;
    }
    if (!run) return;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
    {   // zero this view's status words for the passes that run (16-byte stores)
        uint4 *st = reinterpret_cast<uint4 *>(ws.sort_counts);
        const int64_t per = ws.sort_tiles_cap * kBins / 4, used = c.ntiles * kBins / 4;
        for (int p = 0; p < c.passes; ++p)
            for (int64_t k = gtid; k < used; k += gsz) st[p * per + k] = make_uint4(0u, 0u, 0u, 0u);
    }
    const unsigned long long *__restrict__ keys = ws.keys[0];
    const int hw = (threadIdx.x >> 5) % kHistWarps;
    constexpr int kH = 8;   // keys in flight per thread
    for (int p0 = 0; p0 < c.passes; p0 += 4) {   // 4 passes per read of the keys
        const int np = c.passes - p0 < 4 ? c.passes - p0 : 4;
        for (int k = threadIdx.x; k < kHistWarps * 4 * kBins; k += kBlock) (&h[0][0][0])[k] = 0u;
        __syncthreads();
        for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x * kH + threadIdx.x; i0 < c.e;
             i0 += gsz * kH) {
            unsigned long long key[kH];
#pragma unroll
            for (int q = 0; q < kH; ++q) {
                const int64_t i = i0 + (int64_t)q * blockDim.x;
                key[q] = i < c.e ? keys[i] : 0ull;
            }
#pragma unroll
            for (int q = 0; q < kH; ++q) {
                if (i0 + (int64_t)q * blockDim.x >= c.e) break;
                for (int p = 0; p < np; ++p)
                    atomicAdd(&h[hw][p][digit_of(key[q], c.dmin, c.dtop, c.dbits, c.rbits * (p0 + p),
                                                  c.nbins - 1)], 1u);
            }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < np * kBins; k += kBlock) {
            unsigned cnt = 0;
#pragma unroll
            for (int w = 0; w < kHistWarps; ++w) cnt += (&h[w][0][0])[k];
            if (cnt) atomicAdd(&ws.hist[p0 * kBins + k], cnt);
        }
        __syncthreads();
    }
}

// Exclusive count of digit d over tiles [0, tile): decoupled look-back.  The
// immediate predecessor is read alone first (usually already inclusive); then
// kProbe predecessors per round trip.
__device__ __forceinline__ unsigned look_back(const unsigned *status, int64_t tile, int d) {
    unsigned excl = 0;
    int64_t j = tile - 1;
    unsigned w0 = ld_relaxed_u32(status + j * kBins + d);
    while (!(w0 & ~kCntMask)) w0 = ld_relaxed_u32(status + j * kBins + d);
    excl = w0 & kCntMask;
    if ((w0 & ~kCntMask) == kInc || j == 0) return excl;
    --j;
    while (true) {
        unsigned w[kProbe];
#pragma unroll
        for (int q = 0; q < kProbe; ++q)
            w[q] = j - q >= 0 ? ld_relaxed_u32(status + (j - q) * kBins + d) : kInc;
        int adv = kProbe;
        bool stop = false;
#pragma unroll
        for (int q = 0; q < kProbe; ++q) {
            if (stop) continue;
            const unsigned fl = w[q] & ~kCntMask;
            if (!fl) {   // not yet published: re-poll from here
                adv = q;
                stop = true;
                continue;
            }
            excl += w[q] & kCntMask;
            if (fl == kInc) return excl;
        }
        j -= adv;
    }
}

constexpr int kOsWarps = kSortThreads / 32;

// One CTA of 256 threads per 2048-key tile (64 registers, so 4 CTAs share an
// SM and one CTA's look-back wait overlaps the others' loads and ranking):
// 8 warps rank their 256 keys each into per-warp 16-bit digit counters; each
// thread then owns two digits for the prefix over warps, the status publish
// and the look-back.
#ifndef G6R_SORT_MINB
#define G6R_SORT_MINB 4
#endif
__global__ void __launch_bounds__(kSortThreads, G6R_SORT_MINB)
k_onesweep(const __grid_constant__ Batch b, int tbits, int vbits, int pass, int64_t splat_n) {
    __shared__ unsigned s_goff[kBins];
    __shared__ unsigned short s_wh[kOsWarps][kBins];
    __shared__ unsigned s_base[kBins];
    __shared__ unsigned s_scan[kOsWarps];
    __shared__ long long s_tile;
    const int v = blockIdx.y;
    PassCtx c;
    if (!pass_ctx(b, v, tbits, vbits, pass, c, splat_n)) return;
    const Workspace &ws = b.ws[v];
    const int src = pass_src(pass);
    const bool need_vals = !c.packed || pass == 0;   // packed passes >= 1 move items only
    const unsigned long long *__restrict__ kin = ws.keys[src];
    const unsigned *__restrict__ vin = ws.vals[src];
    unsigned long long *__restrict__ kout = ws.keys[src ^ 1];
    unsigned *__restrict__ vout = ws.vals[src ^ 1];
    unsigned *status = ws.sort_counts + (int64_t)pass * ws.sort_tiles_cap * kBins;
    const unsigned *totals = ws.hist + pass * kBins;
    unsigned long long *ticket = reinterpret_cast<unsigned long long *>(&ws.internal[kTicketSortBase + pass]);
    const int shift = c.rbits * pass;
    const unsigned nbins = c.nbins, dmask = nbins - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kOwn = kBins / kSortThreads;   // digits per thread
    {   // global exclusive digit offsets: thread t owns digits kOwn*t ..
        unsigned cnt[kOwn], cc = 0;
#pragma unroll
        for (int q = 0; q < kOwn; ++q) cc += (cnt[q] = totals[kOwn * tid + q]);
        const unsigned inc = warp_inclusive_scan(cc);
        if (lane == 31) s_scan[warp] = inc;
        __syncthreads();
        unsigned pre = 0;
        for (int w = 0; w < warp; ++w) pre += s_scan[w];
        unsigned run = pre + inc - cc;
#pragma unroll
        for (int q = 0; q < kOwn; ++q) {
            s_goff[kOwn * tid + q] = run;
            run += cnt[q];
        }
    }
    const unsigned lanemask_lt = (1u << lane) - 1u;
    while (true) {
        if (tid == 0) s_tile = (long long)atomicAdd(ticket, 1ull);
        for (int k = tid; k < kOsWarps * kBins / 2; k += kSortThreads)
            reinterpret_cast<unsigned *>(&s_wh[0][0])[k] = 0u;
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= c.ntiles) break;
        // warp w owns the contiguous items [w*256, w*256+256) of the tile, striped
        const int64_t base = tile * kSortTile + (int64_t)warp * (32 * kSortItems);
        unsigned long long key[kSortItems];
        unsigned val[kSortItems];
        unsigned dr[kSortItems];   // digit << 16 | rank within the warp
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * 32 + lane;
            const bool valid = idx < c.e;
            key[k] = valid ? kin[idx] : ~0ull;
            val[k] = (valid && need_vals) ? (c.splat ? (unsigned)idx : vin[idx]) : 0u;
        }
        if (c.packed && pass == 0) {
#pragma unroll
            for (int k = 0; k < kSortItems; ++k) key[k] = pack_entry(key[k], val[k], c);
        }
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * 32 + lane;
            const unsigned d = idx >= c.e ? nbins
                               : c.packed ? (unsigned)(key[k] >> (c.vbits + shift)) & dmask
                                          : digit_of(key[k], c.dmin, c.dtop, c.dbits, shift, dmask);
            const unsigned peers = match_digit(d, c.rbits);
            const int leader = __ffs(peers) - 1;
            unsigned old = 0;
            if (d < nbins && lane == leader) {
                old = s_wh[warp][d];
                s_wh[warp][d] = (unsigned short)(old + (unsigned)__popc(peers));
            }
            old = __shfl_sync(0xffffffffu, old, leader);
            dr[k] = d << 16 | (old + (unsigned)__popc(peers & lanemask_lt));
            __syncwarp();
        }
        __syncthreads();
        unsigned tot[kOwn];
#pragma unroll
        for (int q = 0; q < kOwn; ++q) {   // exclusive prefix over warps, publish
            const int d = tid + q * kSortThreads;
            tot[q] = 0;
            if ((unsigned)d >= nbins) continue;
            unsigned run = 0;
#pragma unroll
            for (int w = 0; w < kOsWarps; ++w) {
                const unsigned cnt = s_wh[w][d];
                s_wh[w][d] = (unsigned short)run;
                run += cnt;
            }
            tot[q] = run;
            st_relaxed_u32(status + tile * kBins + d, (tile == 0 ? kInc : kAgg) | run);
        }
#pragma unroll
        for (int q = 0; q < kOwn; ++q) {   // look back
            const int d = tid + q * kSortThreads;
            if ((unsigned)d >= nbins) continue;
            unsigned excl = 0;
            if (tile > 0) {
                excl = look_back(status, tile, d);
                st_relaxed_u32(status + tile * kBins + d, kInc | (excl + tot[q]));
            }
            s_base[d] = s_goff[d] + excl;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const unsigned d = dr[k] >> 16;
            if (d >= nbins) continue;
            const unsigned pos = s_base[d] + s_wh[warp][d] + (dr[k] & 0xffffu);
            G6R_CHECK((int64_t)pos < c.e);
            kout[pos] = key[k];
            if (!c.packed) vout[pos] = val[k];
        }
        __syncthreads();
    }
}

// Ascending in-place sort of a run of equal-key values (shell sort: runs are
// almost always 2-3 long; a degenerate axis-aligned view can make long ones).
template <typename T>
__device__ void sort_run(T *v, int n) {
    int gap = 1;
    while (gap < n / 3) gap = 3 * gap + 1;
    for (; gap > 0; gap /= 3)
        for (int a = gap; a < n; ++a) {
            const T x = v[a];
            int c = a;
            while (c >= gap && v[c - gap] > x) {
                v[c] = v[c - gap];
                c -= gap;
            }
            v[c] = x;
        }
}

// grid y = view: tile_starts from the boundaries of the sorted keys, the
// row-order fix-up of equal-key runs, and (packed mode) the entry values
// unpacked into vals[0] for the compositor.
__global__ void __launch_bounds__(kBlock)
k_ranges(const __grid_constant__ Batch b, int tbits, int vbits) {
    const int v = blockIdx.y;
    const Workspace &ws = b.ws[v];
    const ViewOut &out = b.out[v];
    const int64_t n_tiles = (int64_t)b.vp[v].tiles_x * b.vp[v].tiles_y;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
    int64_t *starts = ws.tile_starts;
    int64_t *starts2 = out.tile_starts;
    PassCtx c;
    if (!pass_ctx(b, v, tbits, vbits, 0, c)) {
        if (!entries_valid(out.counters, ws.entry_capacity, c.e)) {   // overflow: empty runs
            for (int64_t t = gtid; t <= n_tiles; t += gsz) {
                starts[t] = 0;
                if (starts2) starts2[t] = 0;
            }
            return;
        }
        c.passes = 0;   // nothing to sort (no entries): the raw buffers are the result
        c.packed = false;
    }
    const int64_t e = c.e;
    const bool packed = c.packed;
    const int kshift = packed ? c.vbits : 0;             // item >> kshift = sort key
    const int tshift = packed ? c.dbits + c.vbits : 32;  // item >> tshift = tile
    const unsigned long long vmask = packed ? (1ull << c.vbits) - 1ull : 0ull;
    unsigned long long *keys = ws.keys[c.passes & 1];
    unsigned *vals = ws.vals[packed ? 0 : (c.passes & 1)];
    int32_t *entry_out = out.entry_splat;
    constexpr int kR = 4;   // consecutive entries per thread per step (loads in flight)
    for (int64_t i0 = gtid * kR; i0 <= e; i0 += gsz * kR) {
        unsigned long long k[kR + 2];   // keys[i0-1 .. i0+kR]
#pragma unroll
        for (int q = 0; q < kR + 2; ++q) {
            const int64_t i = i0 - 1 + q;
            k[q] = (i >= 0 && i < e) ? keys[i] : ~0ull;
        }
#pragma unroll
        for (int q = 1; q <= kR; ++q) {
            const int64_t i = i0 - 1 + q;
            if (i > e) break;
            const unsigned long long ki = k[q], kp = k[q - 1];
            const int64_t ti = i < e ? (int64_t)(ki >> tshift) : n_tiles;
            const int64_t tp = i > 0 ? (int64_t)(kp >> tshift) : -1;
            for (int64_t t = tp + 1; t <= ti; ++t) {
                starts[t] = i;
                if (starts2) starts2[t] = i;
            }
            if (i >= e || (i > 0 && (kp >> kshift) == (ki >> kshift))) continue;   // run interior
            // Equal keys (same tile, same f32 depth) must end in row order, the
            // reference's stable tie rule: the chain-free projection emits CTA
            // blocks in completion order, so sort each such run by value.
            int64_t j = i + 1;
            if ((k[q + 1] >> kshift) == (ki >> kshift))
                while (j < e && (keys[j] >> kshift) == (ki >> kshift)) ++j;
            if (packed) {
                if (j - i > 1) sort_run(keys + i, (int)(j - i));   // value bits are the low bits
                for (int64_t m = i; m < j; ++m) {
                    const unsigned val = (unsigned)((m == i && j - i == 1 ? ki : keys[m]) & vmask);
                    vals[m] = val;
                    if (entry_out) entry_out[m] = (int32_t)val;
                }
            } else {
                if (j - i > 1) sort_run(vals + i, (int)(j - i));
                if (entry_out)
                    for (int64_t m = i; m < j; ++m) entry_out[m] = (int32_t)vals[m];
            }
        }
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

static int value_bits(int64_t max_val) {
    int vb = 1;
    while (vb < 31 && (1ll << vb) <= max_val) ++vb;
    return vb;
}

int launch_sort(const Batch &b, int64_t max_val, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    const int64_t n_tiles = (int64_t)b.vp[0].tiles_x * b.vp[0].tiles_y;
    const int tbits = tile_bits(n_tiles);
    const int vbits = value_bits(max_val);
    const int max_passes = sort_passes((int)n_tiles);
    const int sms = num_sms();
    const int64_t tiles_cap = b.ws[0].sort_tiles_cap;
    const unsigned hx = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(b.ws[0].entry_capacity, kBlock), std::max(sms * 4 / b.nviews, 1)));
    k_sort_hist<<<dim3(hx, b.nviews), kBlock, 0, st>>>(b, tbits, vbits, 0);
    trace_mark("sort_hist", st);
    const unsigned ox = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(tiles_cap, std::max<int64_t>(sms * 4 / b.nviews, 1)));
    for (int p = 0; p < max_passes; ++p) {
        k_onesweep<<<dim3(ox, b.nviews), kSortThreads, 0, st>>>(b, tbits, vbits, p, 0);
        trace_mark("onesweep", st);
    }
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

// Splat-level sort: depth radix passes over the n scene rows (the not-drawn
// rows sort last), then the order-preserving tile partition (g6r_tiles.cu).
int launch_splat_sort(const Batch &b, int64_t n, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    if (n == 0) return launch_tile_partition(b, n, 1, st);   // empty runs
    const int vbits = value_bits(n);
    const int max_passes = (32 + 1 + kRadixBits - 1) / kRadixBits;   // depth bits + sentinel
    const int sms = num_sms();
    const unsigned hx = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), kBlock), std::max(sms * 4 / b.nviews, 1)));
    k_sort_hist<<<dim3(hx, b.nviews), kBlock, 0, st>>>(b, 0, vbits, std::max<int64_t>(n, 1));
    trace_mark("sort_hist", st);
    const unsigned ox = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), kSortTile),
                             std::max<int64_t>(sms * 4 / b.nviews, 1)));
    for (int p = 0; p < max_passes; ++p) {
        k_onesweep<<<dim3(ox, b.nviews), kSortThreads, 0, st>>>(b, 0, vbits, p, std::max<int64_t>(n, 1));
        trace_mark("onesweep", st);
    }
    if (cudaGetLastError() != cudaSuccess) return G6R_ECUDA;
    return launch_tile_partition(b, n, vbits, st);
}

int launch_ranges(const Batch &b, int64_t max_val, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    const int64_t cap = b.ws[0].entry_capacity;
    const int64_t n_tiles = (int64_t)b.vp[0].tiles_x * b.vp[0].tiles_y;
    const unsigned gx = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(cap + 1, kBlock), std::max(num_sms() * 4 / b.nviews, 1)));
    k_ranges<<<dim3(gx, b.nviews), kBlock, 0, st>>>(b, tile_bits(n_tiles), value_bits(max_val));
    trace_mark("ranges", st);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
