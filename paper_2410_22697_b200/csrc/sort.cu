// sort.cu -- segmented, stable LSD radix sort of (u64 key, u32 value) pairs:
// one upfront histogram of every digit, one bin scan that also plans the
// passes, then per 8-bit digit a count launch (per-tile digit counts) and a
// scatter launch (each tile sums the counts of the earlier tiles -- independent
// loads, no tile-to-tile look-back chain -- ranks its keys stably and
// scatters), and a final fix-up: 3 + 2 * passes launches.  The element count
// lives on the device; every kernel loops over the tiles that count needs, a
// digit that is the same for every key is skipped (the identity for a stable
// sort), and the fix-up copies the result back to the primary buffers after an
// odd number of executed passes.//
// Used for every total order the method needs:
//   * buffer init: halo by (deg_in desc, id asc)            (R#10)
//   * epoch order: train ids by (Philox key asc, id asc)     (R#8)
//   * eviction:    E by (S_E asc, id asc), R by (S_A desc, deg_in desc, id asc)  (R#16-#18)
// Ties fall back to input order (stability); every caller feeds items in
// ascending-id order, which realises the "id asc" tie-break.
// Segments (independent arrays with device-side lengths) run side by side
// along gridDim.y.
#include <algorithm>
#include <cstdlib>

#include "launch.h"

namespace mgnn {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048
constexpr int kRadix = 256;

// Small sorts (device-side n <= kSmallN, e.g. an eviction round's candidates) use 512-key tiles (2 keys
// per thread): four times the blocks per pass, a quarter of the serial ranking rounds per block -- a
// pass over a few ten thousand keys is bound by one tile's latency, not by bandwidth.
constexpr int kSmallItems = 2;
constexpr int kSmallTile = kSortThreads * kSmallItems;   // 512
constexpr int64_t kSmallN = 65536;

static inline int64_t sort_tiles(int64_t n_max) {
    int64_t t = (n_max + kSortTile - 1) / kSortTile;
    const int64_t ts = (std::min<int64_t>(n_max, kSmallN) + kSmallTile - 1) / kSmallTile;   // small-mode tiles
    t = std::max(t, ts);
    return t < 1 ? 1 : t;
}

// scratch layout:
//   bins   u32 [n_seg][passes][256]            digit histograms -> bin offsets      } zeroed by one
//   plan   i32 [n_seg][passes + 1]             per pass: input parity, or -1 = the  } small memset
//                                              pass is trivial (one digit value holds every key);
//                                              [passes] = parity of the result
//   tcount u32 [n_seg][passes][tiles][256]     per-tile digit counts of each pass (written by
//                                              k_sort_count for the tiles the device-side length uses)
// Every kernel loops over the tiles the device-side length needs (grids of at most a few blocks per
// SM), so a sort sized for n_max that holds a few thousand keys costs a few microseconds a launch.
static size_t head_bytes(int n_seg, int passes) {
    size_t b = (size_t)n_seg * passes * kRadix * 4 + (size_t)n_seg * (passes + 1) * 4 + 4;   // + barrier word
    return (b + 255) / 256 * 256;
}

size_t radix_scratch_bytes(int n_seg, int64_t n_max, int max_passes) {
    const int64_t passes = max_passes, tiles = sort_tiles(n_max);
    return head_bytes(n_seg, (int)passes) + (size_t)n_seg * passes * tiles * kRadix * 4;
}

struct SortScr {
    uint32_t* bins;
    int32_t* plan;
    uint32_t* status;
};

static SortScr carve(void* base, int n_seg, int passes) {
    SortScr s;
    s.bins = (uint32_t*)base;
    s.plan = (int32_t*)(s.bins + (size_t)n_seg * passes * kRadix);
    s.status = (uint32_t*)((char*)base + head_bytes(n_seg, passes));
    return s;
}

// ---- 1. histogram of every digit position in one read of the keys
__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const SortSeg* __restrict__ segs, int passes,
                                                            int64_t tiles_max, SortScr scr) {
    pdl_enter();
    __shared__ uint32_t h[8][kRadix];
    const SortSeg sg = segs[blockIdx.y];
    const int64_t n = *sg.n;
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    for (int p = 0; p < passes; ++p) h[p][threadIdx.x] = 0;
    __syncthreads();
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t base = t * kSortTile;
#pragma unroll
        for (int i = 0; i < kSortItems; ++i) {
            const int64_t idx = base + (int64_t)i * kSortThreads + threadIdx.x;
            if (idx < n) {
                const unsigned long long k = sg.keys[idx];
                for (int p = 0; p < sg.npass; ++p) atomicAdd(&h[p][(unsigned)(k >> sg.shift[p]) & 0xFF], 1u);
            }
        }
    }
    __syncthreads();
    uint32_t* bins = scr.bins + (size_t)blockIdx.y * passes * kRadix;
    for (int p = 0; p < passes; ++p)
        if (h[p][threadIdx.x]) atomicAdd(&bins[p * kRadix + threadIdx.x], h[p][threadIdx.x]);
}

// ---- 2. exclusive scan of each digit histogram -> bin offsets; the pass plan (trivial passes skipped)
__global__ void __launch_bounds__(kSortThreads) k_sort_binscan(const SortSeg* __restrict__ segs, int passes,
                                                               SortScr scr) {
    pdl_enter();
    __shared__ long long sm[8];
    __shared__ int trivial_sh;
    const SortSeg sg = segs[blockIdx.y];
    const long long n = *sg.n;
    uint32_t* bins = scr.bins + (size_t)blockIdx.y * passes * kRadix;
    int32_t* plan = scr.plan + (size_t)blockIdx.y * (passes + 1);
    int parity = 0;
    for (int p = 0; p < passes; ++p) {
        if (threadIdx.x == 0) trivial_sh = 0;
        __syncthreads();
        const uint32_t c = bins[p * kRadix + threadIdx.x];
        if ((long long)c == n) trivial_sh = 1;    // every key has this digit: the pass is the identity
        long long tot;
        const long long ex = block_excl_scan256(c, sm, &tot);
        bins[p * kRadix + threadIdx.x] = (uint32_t)ex;
        const bool skip = p >= sg.npass || n == 0 || trivial_sh;
        if (threadIdx.x == 0) plan[p] = skip ? -1 : parity;
        if (!skip) parity ^= 1;
        __syncthreads();
    }
    if (threadIdx.x == 0) plan[passes] = parity;
}

// ---- 3. one digit pass in two launches (no serial look-back chain: a pass sorts at most a few
// hundred thousand keys, where a chain of tile-to-tile waits costs more than a second launch):
//   k_sort_count   per tile: digit counts -> tcount[seg][tile][256]
//   k_sort_scatter per tile: global offset of each digit = bin offset + counts of the earlier tiles
//                  (independent loads, one column per thread), stable local ranks, scatter
template <int ITEMS>
__device__ __forceinline__ void sort_count_body(const SortSeg& sg, int s, int passes, int p, int parity, int64_t n,
                                                int64_t tiles_max, const SortScr& scr, uint32_t* h) {
    constexpr int kTile = kSortThreads * ITEMS;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const unsigned long long* kin = parity ? sg.keys_tmp : sg.keys;
    const int shift = sg.shift[p];
    const int lane = threadIdx.x & 31;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        h[threadIdx.x] = 0;
        __syncthreads();
        const int64_t base = t * kTile;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int64_t idx = base + (int64_t)i * kSortThreads + threadIdx.x;
            const unsigned digit = idx < n ? ((unsigned)(kin[idx] >> shift) & 0xFF) : (0x100u | lane);
            const unsigned peers = __match_any_sync(kFull, digit);
            if (digit < 0x100u && lane == __ffs(peers) - 1) atomicAdd(&h[digit], (unsigned)__popc(peers));
        }
        __syncthreads();
        scr.status[((size_t)(s * passes + p) * tiles_max + t) * kRadix + threadIdx.x] = h[threadIdx.x];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kSortThreads) k_sort_count(const SortSeg* __restrict__ segs, int passes, int p,
                                                             int64_t tiles_max, SortScr scr) {
    pdl_enter();
    __shared__ uint32_t h[kRadix];
    const int s = blockIdx.y;
    const SortSeg sg = segs[s];
    const int parity = scr.plan[(size_t)s * (passes + 1) + p];
    if (parity < 0) return;
    const int64_t n = *sg.n;
    if (n <= kSmallN)
        sort_count_body<kSmallItems>(sg, s, passes, p, parity, n, tiles_max, scr, h);
    else
        sort_count_body<kSortItems>(sg, s, passes, p, parity, n, tiles_max, scr, h);
}

// Stable local ranks with two block barriers per tile: warp w owns the contiguous items
// [w * 256, (w + 1) * 256) of the tile (8 rounds of 32), ranks them inside the warp against a
// warp-private digit counter row (match_any + __syncwarp only), then one pass over (digit, warp)
// turns the per-warp counts into each warp's offset inside the tile's digit run.
template <int ITEMS>
__device__ __forceinline__ void sort_scatter_body(const SortSeg& sg, int s, int passes, int p, int parity, int64_t n,
                                                  int64_t tiles_max, const SortScr& scr, uint32_t (*wc)[kRadix],
                                                  uint32_t* gofs) {
    constexpr int kTile = kSortThreads * ITEMS;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const unsigned long long* kin = parity ? sg.keys_tmp : sg.keys;
    const uint32_t* vin = parity ? sg.vals_tmp : sg.vals;
    unsigned long long* kout = parity ? sg.keys : sg.keys_tmp;
    uint32_t* vout = parity ? sg.vals : sg.vals_tmp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int shift = sg.shift[p];
    const uint32_t* tc = scr.status + ((size_t)(s * passes + p) * tiles_max) * kRadix;
    constexpr int kPerWarp = kTile / 8;        // ITEMS * 32 items per warp
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * kTile + (int64_t)warp * kPerWarp;
        unsigned long long key[ITEMS];
        uint32_t val[ITEMS], rank[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {              // every load of the tile in flight at once
            const int64_t idx = base + i * 32 + lane;
            key[i] = idx < n ? kin[idx] : 0ull;
            val[i] = idx < n ? vin[idx] : 0u;
        }
        {   // thread d: exclusive prefix of digit d over the earlier tiles (independent loads)
            const int d = threadIdx.x;
            uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            int64_t j = 0;
            for (; j + 4 <= tile; j += 4) {
                a0 += tc[(size_t)j * kRadix + d];
                a1 += tc[(size_t)(j + 1) * kRadix + d];
                a2 += tc[(size_t)(j + 2) * kRadix + d];
                a3 += tc[(size_t)(j + 3) * kRadix + d];
            }
            for (; j < tile; ++j) a0 += tc[(size_t)j * kRadix + d];
            gofs[d] = scr.bins[(size_t)(s * passes + p) * kRadix + d] + a0 + a1 + a2 + a3;
        }
        for (int d = lane; d < kRadix; d += 32) wc[warp][d] = 0;     // the warp's own counter row
        __syncwarp();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const bool valid = base + i * 32 + lane < n;
            const unsigned digit = valid ? ((unsigned)(key[i] >> shift) & 0xFF) : (0x100u | lane);
            const unsigned peers = __match_any_sync(kFull, digit);
            const unsigned r = __popc(peers & lt);
            rank[i] = valid ? wc[warp][digit & 0xFF] + r : 0xFFFFFFFFu;
            __syncwarp();
            if (valid && r == 0) wc[warp][digit] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        {   // thread d: each warp's offset inside the tile's run of digit d
            const int d = threadIdx.x;
            uint32_t acc = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const uint32_t c = wc[w][d];
                wc[w][d] = acc;
                acc += c;
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (rank[i] == 0xFFFFFFFFu) continue;
            const unsigned digit = (unsigned)(key[i] >> shift) & 0xFF;
            const uint32_t pos = gofs[digit] + wc[warp][digit] + rank[i];
            MGNN_CHECK(pos < n, "scatter pos=%u n=%lld seg=%d", pos, (long long)n, s);
            kout[pos] = key[i];
            vout[pos] = val[i];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kSortThreads) k_sort_scatter(const SortSeg* __restrict__ segs, int passes, int p,
                                                               int64_t tiles_max, SortScr scr) {
    pdl_enter();
    __shared__ uint32_t wc[8][kRadix];     // per-warp digit counts, then the warp's offset in the digit run
    __shared__ uint32_t gofs[kRadix];      // global offset of the tile's first item of each digit
    const int s = blockIdx.y;
    const SortSeg sg = segs[s];
    const int parity = scr.plan[(size_t)s * (passes + 1) + p];
    if (parity < 0) return;                    // beyond this segment's schedule, or a trivial digit
    const int64_t n = *sg.n;
    if (n <= kSmallN)
        sort_scatter_body<kSmallItems>(sg, s, passes, p, parity, n, tiles_max, scr, wc, gofs);
    else
        sort_scatter_body<kSortItems>(sg, s, passes, p, parity, n, tiles_max, scr, wc, gofs);
}

// ---- 4. an odd number of executed passes left the result in the tmp buffers: copy it back
__global__ void __launch_bounds__(kSortThreads) k_sort_fix(const SortSeg* __restrict__ segs, int passes, SortScr scr) {
    pdl_enter();
    const SortSeg sg = segs[blockIdx.y];
    if (scr.plan[(size_t)blockIdx.y * (passes + 1) + passes] == 0) return;
    const int64_t n = *sg.n;
    for (int64_t i = (int64_t)blockIdx.x * kSortThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kSortThreads) {
        sg.keys[i] = sg.keys_tmp[i];
        sg.vals[i] = sg.vals_tmp[i];
    }
}

// ---- the whole sort in ONE cooperative launch (MGNN_SORT_COOP=1): the same phases separated by grid-wide
// barriers instead of kernel boundaries.  An eviction round sorts a few thousand to a few ten thousand
// candidates, where the 3 + 2 * passes dependent launches cost more than their work (products: ~150 us
// for ~70k keys); here every block takes (segment, tile) pairs in a fixed stride.
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned& gen) {
    // sense-reversal-free barrier on a monotone counter: block b waits until ctr >= (gen + 1) * nblocks
    __syncthreads();
    const unsigned nb = gridDim.x * gridDim.y;
    ++gen;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (true) {
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= gen * nb) break;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSortThreads) k_sort_coop(const SortSeg* __restrict__ segs, int n_seg, int passes,
                                                            int64_t tiles_max, SortScr scr, unsigned* bar) {
    pdl_enter();
    __shared__ uint32_t run[kRadix];
    __shared__ uint32_t wc[8][kRadix];
    __shared__ uint32_t gofs[kRadix];
    __shared__ uint32_t h8[8][kRadix];
    __shared__ long long sm[8];
    __shared__ int trivial_sh;
    unsigned gen = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t nblk = gridDim.x;
    const int64_t work = (int64_t)n_seg * tiles_max;      // (segment, tile) pairs, segment-major
    // ---- histogram of every digit position
    for (int p = 0; p < passes; ++p) h8[p][threadIdx.x] = 0;
    int cur_seg = -1;
    auto flush_hist = [&]() {
        __syncthreads();
        if (cur_seg >= 0) {
            uint32_t* bins = scr.bins + (size_t)cur_seg * passes * kRadix;
            for (int p = 0; p < passes; ++p) {
                if (h8[p][threadIdx.x]) atomicAdd(&bins[p * kRadix + threadIdx.x], h8[p][threadIdx.x]);
                h8[p][threadIdx.x] = 0;
            }
        }
        __syncthreads();
    };
    for (int64_t wi = blockIdx.x; wi < work; wi += nblk) {
        const int sgi = (int)(wi / tiles_max);
        const int64_t t = wi - (int64_t)sgi * tiles_max;
        const SortSeg sg = segs[sgi];
        const int64_t n = *sg.n;
        if (t * kSortTile >= n) continue;
        if (sgi != cur_seg) {
            flush_hist();
            cur_seg = sgi;
        }
#pragma unroll
        for (int i = 0; i < kSortItems; ++i) {
            const int64_t idx = t * kSortTile + (int64_t)i * kSortThreads + threadIdx.x;
            if (idx < n) {
                const unsigned long long k = sg.keys[idx];
                for (int p = 0; p < sg.npass; ++p) atomicAdd(&h8[p][(unsigned)(k >> sg.shift[p]) & 0xFF], 1u);
            }
        }
    }
    flush_hist();
    grid_barrier(bar, gen);
    // ---- bin offsets and the pass plan (block sgi < n_seg)
    for (int sgi = blockIdx.x; sgi < n_seg; sgi += nblk) {
        const SortSeg sg = segs[sgi];
        const long long n = *sg.n;
        uint32_t* bins = scr.bins + (size_t)sgi * passes * kRadix;
        int32_t* plan = scr.plan + (size_t)sgi * (passes + 1);
        int parity = 0;
        for (int p = 0; p < passes; ++p) {
            if (threadIdx.x == 0) trivial_sh = 0;
            __syncthreads();
            const uint32_t c = bins[p * kRadix + threadIdx.x];
            if ((long long)c == n) trivial_sh = 1;
            long long tot;
            const long long ex = block_excl_scan256(c, sm, &tot);
            bins[p * kRadix + threadIdx.x] = (uint32_t)ex;
            const bool skip = p >= sg.npass || n == 0 || trivial_sh;
            if (threadIdx.x == 0) plan[p] = skip ? -1 : parity;
            if (!skip) parity ^= 1;
            __syncthreads();
        }
        if (threadIdx.x == 0) plan[passes] = parity;
        __syncthreads();
    }
    grid_barrier(bar, gen);
    // ---- passes: per-tile counts | barrier | prefix over earlier tiles, stable ranks, scatter | barrier
    for (int p = 0; p < passes; ++p) {
        for (int64_t wi = blockIdx.x; wi < work; wi += nblk) {
            const int sgi = (int)(wi / tiles_max);
            const int64_t t = wi - (int64_t)sgi * tiles_max;
            const SortSeg sg = segs[sgi];
            const int parity = scr.plan[(size_t)sgi * (passes + 1) + p];
            const int64_t n = *sg.n;
            if (parity < 0 || t * kSortTile >= n) continue;
            const unsigned long long* kin = parity ? sg.keys_tmp : sg.keys;
            const int shift = sg.shift[p];
            run[threadIdx.x] = 0;
            __syncthreads();
            unsigned long long kk[kSortItems];
#pragma unroll
            for (int i = 0; i < kSortItems; ++i) {
                const int64_t idx = t * kSortTile + (int64_t)i * kSortThreads + threadIdx.x;
                kk[i] = idx < n ? kin[idx] : 0ull;
            }
#pragma unroll
            for (int i = 0; i < kSortItems; ++i) {
                const int64_t idx = t * kSortTile + (int64_t)i * kSortThreads + threadIdx.x;
                const unsigned digit = idx < n ? ((unsigned)(kk[i] >> shift) & 0xFF) : (0x100u | lane);
                const unsigned peers = __match_any_sync(kFull, digit);
                if (digit < 0x100u && lane == __ffs(peers) - 1) atomicAdd(&run[digit], (unsigned)__popc(peers));
            }
            __syncthreads();
            scr.status[((size_t)(sgi * passes + p) * tiles_max + t) * kRadix + threadIdx.x] = run[threadIdx.x];
            __syncthreads();
        }
        grid_barrier(bar, gen);
        for (int64_t wi = blockIdx.x; wi < work; wi += nblk) {
            const int sgi = (int)(wi / tiles_max);
            const int64_t tile = wi - (int64_t)sgi * tiles_max;
            const SortSeg sg = segs[sgi];
            const int parity = scr.plan[(size_t)sgi * (passes + 1) + p];
            const int64_t n = *sg.n;
            if (parity < 0 || tile * kSortTile >= n) continue;
            const unsigned long long* kin = parity ? sg.keys_tmp : sg.keys;
            const uint32_t* vin = parity ? sg.vals_tmp : sg.vals;
            unsigned long long* kout = parity ? sg.keys : sg.keys_tmp;
            uint32_t* vout = parity ? sg.vals : sg.vals_tmp;
            const int shift = sg.shift[p];
            const uint32_t* tc = scr.status + ((size_t)(sgi * passes + p) * tiles_max) * kRadix;
            {
                const int d = threadIdx.x;
                uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                int64_t j = 0;
                for (; j + 4 <= tile; j += 4) {
                    a0 += tc[(size_t)j * kRadix + d];
                    a1 += tc[(size_t)(j + 1) * kRadix + d];
                    a2 += tc[(size_t)(j + 2) * kRadix + d];
                    a3 += tc[(size_t)(j + 3) * kRadix + d];
                }
                for (; j < tile; ++j) a0 += tc[(size_t)j * kRadix + d];
                gofs[d] = scr.bins[(size_t)(sgi * passes + p) * kRadix + d] + a0 + a1 + a2 + a3;
                run[d] = 0;
                for (int w = 0; w < 8; ++w) wc[w][d] = 0;
            }
            __syncthreads();
            unsigned long long key[kSortItems];
            uint32_t val[kSortItems], rank[kSortItems];
#pragma unroll
            for (int i = 0; i < kSortItems; ++i) {     // every load of the tile in flight at once
                const int64_t idx = tile * kSortTile + (int64_t)i * kSortThreads + threadIdx.x;
                key[i] = idx < n ? kin[idx] : 0ull;
                val[i] = idx < n ? vin[idx] : 0u;
            }
#pragma unroll
            for (int i = 0; i < kSortItems; ++i) {
                const int64_t idx = tile * kSortTile + (int64_t)i * kSortThreads + threadIdx.x;
                const bool valid = idx < n;
                const unsigned digit = valid ? ((unsigned)(key[i] >> shift) & 0xFF) : (0x100u | lane);
                const unsigned peers = __match_any_sync(kFull, digit);
                const unsigned r = __popc(peers & lt);
                if (valid && r == 0) wc[warp][digit] = __popc(peers);
                __syncthreads();
                {
                    uint32_t acc = run[threadIdx.x];
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        const uint32_t c = wc[w][threadIdx.x];
                        wc[w][threadIdx.x] = acc;
                        acc += c;
                    }
                    run[threadIdx.x] = acc;
                }
                __syncthreads();
                rank[i] = valid ? wc[warp][digit] + r : 0xFFFFFFFFu;
                __syncthreads();
                for (int w = 0; w < 8; ++w) wc[w][threadIdx.x] = 0;
                __syncthreads();
            }
#pragma unroll
            for (int i = 0; i < kSortItems; ++i) {
                if (rank[i] == 0xFFFFFFFFu) continue;
                const unsigned digit = (unsigned)(key[i] >> shift) & 0xFF;
                const uint32_t pos = gofs[digit] + rank[i];
                kout[pos] = key[i];
                vout[pos] = val[i];
            }
            __syncthreads();
        }
        grid_barrier(bar, gen);
    }
    // ---- fix-up: an odd number of executed passes left the result in the tmp buffers
    for (int sgi = 0; sgi < n_seg; ++sgi) {
        if (scr.plan[(size_t)sgi * (passes + 1) + passes] == 0) continue;
        const SortSeg sg = segs[sgi];
        const int64_t n = *sg.n;
        for (int64_t i = (int64_t)blockIdx.x * kSortThreads + threadIdx.x; i < n; i += nblk * kSortThreads) {
            sg.keys[i] = sg.keys_tmp[i];
            sg.vals[i] = sg.vals_tmp[i];
        }
    }
}

void radix_sort_pairs(const SortSeg* segs_dev, int n_seg, int64_t n_max, int max_passes, void* scratch,
                      cudaStream_t s) {
    if (n_seg < 1) return;
    const int passes = max_passes;
    const int64_t tiles = sort_tiles(n_max);
    cudaMemsetAsync(scratch, 0, head_bytes(n_seg, passes), s);
    const SortScr scr = carve(scratch, n_seg, passes);
    // grids of at most ~4 blocks per SM over all segments; every kernel loops over its tiles
    int64_t gx = ((int64_t)num_sms() * 4 + n_seg - 1) / n_seg;
    if (gx > tiles) gx = tiles;
    dim3 grid((unsigned)(gx < 1 ? 1 : gx), (unsigned)n_seg);
    // MGNN_SORT_COOP=1: the single cooperative launch below (measured slower on products' eviction
    // rounds: 180 vs 150 us per sort -- the passes' work, not the launches, dominates)
    static const int coop = [] {
        const char* e = getenv("MGNN_SORT_COOP");
        return e ? atoi(e) : 0;
    }();
    if (coop) {                               // one cooperative launch, 1 block per SM at most
        int64_t nb = std::min<int64_t>((int64_t)num_sms(), (int64_t)n_seg * tiles);
        if (nb < 1) nb = 1;
        unsigned* bar = reinterpret_cast<unsigned*>(scr.plan + (size_t)n_seg * (passes + 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)nb);
        cfg.blockDim = dim3(kSortThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, k_sort_coop, segs_dev, n_seg, passes, tiles, scr, bar) == cudaSuccess) {
            count_launches(1, __func__, s);
            return;
        }
        cudaGetLastError();                   // fall back to the multi-launch sort below
    }
    launch_k(k_sort_hist, grid, dim3(kSortThreads), 0, s, segs_dev, passes, tiles, scr);
    launch_k(k_sort_binscan, dim3(1, n_seg), dim3(kSortThreads), 0, s, segs_dev, passes, scr);
    for (int p = 0; p < passes; ++p) {
        launch_k(k_sort_count, grid, dim3(kSortThreads), 0, s, segs_dev, passes, p, tiles, scr);
        launch_k(k_sort_scatter, grid, dim3(kSortThreads), 0, s, segs_dev, passes, p, tiles, scr);
    }
    launch_k(k_sort_fix, grid, dim3(kSortThreads), 0, s, segs_dev, passes, scr);
    count_launches(3 + 2 * passes, __func__, s);
}

}  // namespace mgnn
