// sort.cu -- segmented, stable LSD radix sort of (u64 key, u32 value) pairs
// ("onesweep" structure: one upfront histogram of every digit, one bin scan,
// then one scatter launch per 8-bit digit whose tiles find their global digit
// offsets by a decoupled look-back -- 2 + passes launches per sort instead of
// 3 per pass).
//
// Used for every total order the method needs:
//   * buffer init: halo by (deg_in desc, id asc)            (R#10)
//   * epoch order: train ids by (Philox key asc, id asc)     (R#8)
//   * eviction:    E by (S_E asc, id asc), R by (S_A desc, deg_in desc, id asc)  (R#16-#18)
// Ties fall back to input order (stability); every caller feeds items in
// ascending-id order, which realises the "id asc" tie-break.
// Segments (independent arrays with device-side lengths) run side by side
// along gridDim.y.
#include "launch.h"

namespace mgnn {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048
constexpr int kRadix = 256;

static inline int64_t sort_tiles(int64_t n_max) {
    int64_t t = (n_max + kSortTile - 1) / kSortTile;
    return t < 1 ? 1 : t;
}

// scratch layout (all zeroed by one memset per sort):
//   bins   u32 [n_seg][passes][256]            digit histograms -> bin offsets
//   ctr    i32 [n_seg][passes]                 dynamic tile ids
//   status u32 [n_seg][passes][tiles][256]     look-back words: [31:30] flag, [29:0] count
size_t radix_scratch_bytes(int n_seg, int64_t n_max, int max_passes) {
    const int64_t passes = max_passes, tiles = sort_tiles(n_max);
    size_t b = (size_t)n_seg * passes * kRadix * 4;
    b += (size_t)n_seg * passes * 4;
    b = (b + 255) / 256 * 256;
    b += (size_t)n_seg * passes * tiles * kRadix * 4;
    return b;
}

struct SortScr {
    uint32_t* bins;
    int32_t* ctr;
    uint32_t* status;
};

static SortScr carve(void* base, int n_seg, int passes) {
    SortScr s;
    s.bins = (uint32_t*)base;
    s.ctr = (int32_t*)(s.bins + (size_t)n_seg * passes * kRadix);
    size_t off = (size_t)n_seg * passes * kRadix * 4 + (size_t)n_seg * passes * 4;
    off = (off + 255) / 256 * 256;
    s.status = (uint32_t*)((char*)base + off);
    return s;
}

// ---- 1. histogram of every digit position in one read of the keys
__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const SortSeg* __restrict__ segs, int passes,
                                                            SortScr scr) {
    __shared__ uint32_t h[8][kRadix];
    const SortSeg sg = segs[blockIdx.y];
    const int64_t n = *sg.n;
    for (int p = 0; p < passes; ++p) h[p][threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    if (base < n) {
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

// ---- 2. exclusive scan of each digit histogram -> bin offsets
__global__ void __launch_bounds__(kSortThreads) k_sort_binscan(int passes, SortScr scr) {
    __shared__ long long sm[8];
    uint32_t* bins = scr.bins + (size_t)blockIdx.y * passes * kRadix;
    for (int p = 0; p < passes; ++p) {
        long long tot;
        const long long ex = block_excl_scan256(bins[p * kRadix + threadIdx.x], sm, &tot);
        bins[p * kRadix + threadIdx.x] = (uint32_t)ex;
    }
}

__device__ __forceinline__ void st_rel32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acq32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
constexpr uint32_t kSAgg = 1u << 30, kSInc = 2u << 30, kSMask = (1u << 30) - 1;

// ---- 3. one digit pass: local stable ranks, per-digit look-back, scatter
__global__ void __launch_bounds__(kSortThreads) k_sort_pass(const SortSeg* __restrict__ segs, int passes, int p,
                                                            int64_t tiles_max, SortScr scr) {
    __shared__ uint32_t run[kRadix];       // per-digit running count inside the tile
    __shared__ uint32_t wc[8][kRadix];     // per-warp digit counts of the current round
    __shared__ uint32_t gofs[kRadix];      // global offset of the tile's first item of each digit
    __shared__ int tslot;
    const int s = blockIdx.y;
    const SortSeg sg = segs[s];
    if (p >= sg.npass) return;                 // this segment's schedule has fewer digits
    const int64_t n = *sg.n;
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    const int tile = claim_tile(scr.ctr + s * passes + p, &tslot);
    if (tile >= ntiles) return;
    const int parity = p & 1;
    const unsigned long long* kin = parity ? sg.keys_tmp : sg.keys;
    const uint32_t* vin = parity ? sg.vals_tmp : sg.vals;
    unsigned long long* kout = parity ? sg.keys : sg.keys_tmp;
    uint32_t* vout = parity ? sg.vals : sg.vals_tmp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int shift = sg.shift[p];
    const int64_t base = (int64_t)tile * kSortTile;
    run[threadIdx.x] = 0;
    for (int w = 0; w < 8; ++w) wc[w][threadIdx.x] = 0;
    __syncthreads();
    unsigned long long key[kSortItems];
    uint32_t val[kSortItems], rank[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + (int64_t)i * kSortThreads + threadIdx.x;
        const bool valid = idx < n;
        key[i] = valid ? kin[idx] : 0ull;
        val[i] = valid ? vin[idx] : 0u;
        const unsigned digit = valid ? ((unsigned)(key[i] >> shift) & 0xFF) : (0x100u | lane);
        const unsigned peers = __match_any_sync(kFull, digit);
        const unsigned r = __popc(peers & lt);
        if (valid && r == 0) wc[warp][digit] = __popc(peers);
        __syncthreads();
        {   // per digit: exclusive prefix over warps of this round, advance the tile-local count
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
    {   // thread d: publish the tile's count of digit d, look back for its exclusive prefix
        const int d = threadIdx.x;
        const uint32_t cnt = run[d];
        uint32_t* st = scr.status + ((size_t)(s * passes + p) * tiles_max) * kRadix;
        uint32_t excl = 0;
        if (tile == 0) {
            st_rel32(&st[d], kSInc | cnt);
        } else {
            st_rel32(&st[(size_t)tile * kRadix + d], kSAgg | cnt);
            for (int j = tile - 1; j >= 0; --j) {
                uint32_t v;
                do {
                    v = ld_acq32(&st[(size_t)j * kRadix + d]);
                } while ((v & ~kSMask) == 0);
                excl += v & kSMask;
                if ((v & ~kSMask) == kSInc) break;
            }
            st_rel32(&st[(size_t)tile * kRadix + d], kSInc | (excl + cnt));
        }
        gofs[d] = scr.bins[(size_t)(s * passes + p) * kRadix + d] + excl;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        if (rank[i] == 0xFFFFFFFFu) continue;
        const unsigned digit = (unsigned)(key[i] >> shift) & 0xFF;
        const uint32_t pos = gofs[digit] + rank[i];
        MGNN_CHECK(pos < n, "scatter pos=%u n=%lld seg=%d", pos, (long long)n, s);
        kout[pos] = key[i];
        vout[pos] = val[i];
    }
}

void radix_sort_pairs(const SortSeg* segs_dev, int n_seg, int64_t n_max, int max_passes, void* scratch,
                      cudaStream_t s) {
    if (n_seg < 1) return;
    const int passes = max_passes;
    const int64_t tiles = sort_tiles(n_max);
    cudaMemsetAsync(scratch, 0, radix_scratch_bytes(n_seg, n_max, max_passes), s);
    const SortScr scr = carve(scratch, n_seg, passes);
    dim3 grid((unsigned)tiles, (unsigned)n_seg);
    k_sort_hist<<<grid, kSortThreads, 0, s>>>(segs_dev, passes, scr);
    k_sort_binscan<<<dim3(1, n_seg), kSortThreads, 0, s>>>(passes, scr);
    for (int p = 0; p < passes; ++p) k_sort_pass<<<grid, kSortThreads, 0, s>>>(segs_dev, passes, p, tiles, scr);
    count_launches(2 + passes, __func__, s);
}

}  // namespace mgnn
