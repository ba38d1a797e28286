// sort.cu -- segmented stable LSD radix sort of (u64 key, u32 value) pairs.
//
// Used for every total order the method needs:
//   * buffer init: halo by (deg_in desc, id asc)            (R#10)
//   * epoch order: train ids by (Philox key asc, id asc)     (R#8)
//   * eviction:    E by (S_E asc, id asc), R by (S_A desc, deg_in desc, id asc)  (R#16-#18)
// Ties fall back to input order (stability), and every caller feeds items in
// ascending-id order, which realises the "id asc" tie-break.
//
// Per 8-bit digit pass: (1) per-tile digit histogram, (2) per-segment
// exclusive scan in (digit, tile) order, (3) stable scatter (warp match_any
// ranks + per-warp digit prefix in shared memory).  Segments run side by side
// along gridDim.y.
#include "launch.h"

namespace mgnn {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048
constexpr int kRadix = 256;

static inline int64_t sort_tiles(int64_t n_max) { return (n_max + kSortTile - 1) / kSortTile; }

size_t radix_hist_words(int n_seg, int64_t n_max) {
    int64_t t = sort_tiles(n_max);
    if (t < 1) t = 1;
    return (size_t)n_seg * kRadix * (size_t)t;
}

__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const SortSeg* __restrict__ segs, int64_t tiles_max,
                                                             int shift, int parity, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kRadix];
    const SortSeg sg = segs[blockIdx.y];
    const int64_t n = *sg.n;
    const int64_t tile = blockIdx.x;
    h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long* keys = parity ? sg.keys_tmp : sg.keys;
    const int64_t base = tile * kSortTile;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        int64_t idx = base + (int64_t)i * kSortThreads + threadIdx.x;
        if (idx < n) atomicAdd(&h[(unsigned)(keys[idx] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    hist[((size_t)blockIdx.y * kRadix + threadIdx.x) * tiles_max + tile] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scan(const SortSeg* __restrict__ segs, int64_t tiles_max,
                                                             uint32_t* __restrict__ hist) {
    __shared__ long long sm[8];
    const int64_t n = *segs[blockIdx.y].n;
    const int64_t nt = (n + kSortTile - 1) / kSortTile;
    uint32_t* row = hist + ((size_t)blockIdx.y * kRadix + threadIdx.x) * tiles_max;
    long long sum = 0;
    for (int64_t t = 0; t < nt; ++t) sum += row[t];
    long long total;
    long long run = block_excl_scan256(sum, sm, &total);
    for (int64_t t = 0; t < nt; ++t) {
        uint32_t c = row[t];
        row[t] = (uint32_t)run;
        run += c;
    }
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const SortSeg* __restrict__ segs, int64_t tiles_max,
                                                                int shift, int parity,
                                                                const uint32_t* __restrict__ hist) {
    __shared__ uint32_t run[kRadix];
    __shared__ uint32_t wc[8][kRadix];
    const SortSeg sg = segs[blockIdx.y];
    const int64_t n = *sg.n;
    const int64_t tile = blockIdx.x;
    const int64_t base = tile * kSortTile;
    if (base >= n) return;
    const unsigned long long* kin = parity ? sg.keys_tmp : sg.keys;
    const uint32_t* vin = parity ? sg.vals_tmp : sg.vals;
    unsigned long long* kout = parity ? sg.keys : sg.keys_tmp;
    uint32_t* vout = parity ? sg.vals : sg.vals_tmp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    run[threadIdx.x] = hist[((size_t)blockIdx.y * kRadix + threadIdx.x) * tiles_max + tile];
    for (int w = 0; w < 8; ++w) wc[w][threadIdx.x] = 0;
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + (int64_t)i * kSortThreads + threadIdx.x;
        const bool valid = idx < n;
        unsigned long long key = valid ? kin[idx] : 0ull;
        uint32_t val = valid ? vin[idx] : 0u;
        const unsigned digit = valid ? ((unsigned)(key >> shift) & 0xFF) : (0x100u | lane);
        const unsigned peers = __match_any_sync(kFull, digit);
        const unsigned rank = __popc(peers & lt);
        if (valid && rank == 0) wc[warp][digit] = __popc(peers);
        __syncthreads();
        {   // per digit: exclusive prefix over warps, advance the tile-running offset
            uint32_t acc = run[threadIdx.x];
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                uint32_t c = wc[w][threadIdx.x];
                wc[w][threadIdx.x] = acc;
                acc += c;
            }
            run[threadIdx.x] = acc;
        }
        __syncthreads();
        if (valid) {
            const uint32_t pos = wc[warp][digit] + rank;
            MGNN_CHECK(pos < n, "scatter pos=%u n=%lld seg=%d", pos, (long long)n, (int)blockIdx.y);
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
        for (int w = 0; w < 8; ++w) wc[w][threadIdx.x] = 0;
        __syncthreads();
    }
}

void radix_sort_pairs(const SortSeg* segs_dev, int n_seg, int64_t n_max, int bits, uint32_t* hist, cudaStream_t s) {
    int64_t tiles = sort_tiles(n_max);
    if (tiles < 1 || n_seg < 1) return;
    dim3 grid((unsigned)tiles, (unsigned)n_seg);
    int passes = bits / 8;
    for (int p = 0; p < passes; ++p) {
        int parity = p & 1;
        k_radix_hist<<<grid, kSortThreads, 0, s>>>(segs_dev, tiles, p * 8, parity, hist);
        k_radix_scan<<<dim3(1, n_seg), kSortThreads, 0, s>>>(segs_dev, tiles, hist);
        k_radix_scatter<<<grid, kSortThreads, 0, s>>>(segs_dev, tiles, p * 8, parity, hist);
    }
    count_launches(3 * passes, __func__);
}

}  // namespace mgnn
