// score.cu -- scoreboards and buffer maintenance (§3.2, Alg.2 l.6-9,
// l.12-19, EVICT_AND_REPLACE l.25-34; Alg.1 INITIALIZE_PREFETCHER).
//
// fp32 throughout with explicit round-to-nearest intrinsics and no FTZ
// (DESIGN R#12), so every score is bit-identical to the step-by-step oracle.
//
// Eviction round (every Delta steps, R#14):
//   k_select  order-preserving compaction of E = {buffered, S_E < alpha} and
//             R = {not buffered, S_A >= theta_r} with UNIQUE 64-bit keys
//               E: S_E bits << 32 | node id             -> ascending = (S_E asc, id asc)      (R#16)
//               R: ~S_A bits << 32 | rank_deg            -> ascending = (S_A desc, deg_in desc, id asc) (R#18)
//             (rank_deg = position in the static (deg_in desc, id asc) order of the buffer init;
//             E is scanned in id order, R in that degree order, so each list is in its low word's
//             order), plus a histogram of the top 12 key bits; on eviction windows it also applies
//             the window's decay (k_decay folded in).  K = min(|E|, |R|) (R#19) and, per list, the
//             threshold digit T below which the K smallest keys lie follow from the histograms.
//   small |BUF| (<= kEvMax):
//   k_cand    compacts the candidates (digit <= T) -- typically a few hundred;
//   k_rank    ranks every candidate by counting smaller candidate keys (keys are unique, so the
//             rank IS the sorted position) and writes the K winners in order: no sort at all.
//   large |BUF|: k_hist2 + k_cand_ord (order-preserving), then a stable radix sort (sort.cu) of the
//             candidates' score word only (4 digits) -- K and a bucket instead of the whole lists;
//             MGNN_EV_SELECT=0: unordered candidates from scoreboard scans, all 8 key bytes sorted;
//             MGNN_EVICT_SORT=2 sorts the whole lists instead.
//   k_swap_refill  pair i = (E[i], R[i]): swap of P:224, refill from the owner's table.
#include <algorithm>

#include "launch.h"

namespace mgnn {

constexpr int kSThreads = 256;
constexpr int kDig = 4096;            // 12-bit top-of-key histogram

static inline unsigned blocks_for(int64_t n, int per_block) {
    int64_t b = (n + per_block - 1) / per_block;
    if (b > (int64_t)num_sms() * 8) b = (int64_t)num_sms() * 8;
    return (unsigned)(b < 1 ? 1 : b);
}

// ------------------------------------------------------------------ decay (Alg.2 l.6-9)
// Slot s was hit at popc(mask) of the window's n_steps steps; each other step
// multiplies S_E by gamma once (the same sequence of RN products the paper's
// per-step loop performs: only *gamma ever touches S_E between rounds).
__global__ void __launch_bounds__(kSThreads) k_decay(const PartDev* __restrict__ parts, int n_steps, float gamma,
                                                     const unsigned long long* ovf, uint64_t t_last) {
    pdl_enter();
    if (*ovf <= t_last) return;                  // arena overflow: the window was skipped
    const PartDev& pd = parts[blockIdx.y];
    for (int64_t s = (int64_t)blockIdx.x * kSThreads + threadIdx.x; s < pd.cap; s += (int64_t)gridDim.x * kSThreads) {
        const unsigned long long mask = pd.hitmask[s];
        const int unused = n_steps - __popcll(mask);
        float v = pd.se[s];
        for (int i = 0; i < unused; ++i) v = __fmul_rn(v, gamma);
        pd.se[s] = v;
        if (mask) pd.hitmask[s] = 0ull;
    }
}

void launch_decay(const PartDev* parts, int n_lp, int64_t cap_max, int n_steps, float gamma,
                  const unsigned long long* ovf, uint64_t t_last, cudaStream_t s) {
    if (cap_max < 1) return;
    dim3 grid(blocks_for(cap_max, kSThreads), n_lp);
    launch_k(k_decay, grid, dim3(kSThreads), 0, s, parts, n_steps, gamma, ovf, t_last);
    count_launches(1, __func__, s);
}

// ------------------------------------------------------------------ candidate selection
// Segment 2*lp = E, 2*lp+1 = R; E scanned in halo (= id) order, R in the static (deg_in desc, id asc)
// order of the buffer init, so each list is already in the order of its key's LOW word: a stable sort
// of the high word (the score) alone yields the full key order (k_cand_ord + a 4-digit sort).  Scores here are >= +0, so
// their IEEE bit patterns order like the values.  Order-preserving compaction by a decoupled
// look-back scan, plus a warp-aggregated histogram of key >> 52 per list.
// decay_steps > 0: the window's decay (k_decay) is folded in -- the E scan visits every slot exactly once
// (through its halo node), so it applies the slot's pending gamma products before reading S_E; one
// dependent launch less in the eviction round.
#ifndef MGNN_SEL_ITEMS
#define MGNN_SEL_ITEMS 16
#endif
constexpr int kSelItems = MGNN_SEL_ITEMS;           // list entries per thread (tile = 256 x kSelItems); 16:
                                                    // half the look-back chain, products eviction round -3 %
__global__ void __launch_bounds__(kSThreads) k_select(const PartDev* __restrict__ parts, float alpha, float theta_r,
                                                      const SortSeg* __restrict__ segs, long long* __restrict__ n_out,
                                                      Scratch sc, int64_t tiles_max, EvScratch ev, int decay_steps,
                                                      float gamma, const unsigned long long* ovf, uint64_t t_last) {
    pdl_enter();
    const bool decay = decay_steps > 0 && !(*ovf <= t_last);   // an overflowed window is not decayed
    __shared__ long long sm[8];
    __shared__ int tslot;
    __shared__ long long prefix_sh;
    const int sg = blockIdx.y;
    const PartDev& pd = parts[sg >> 1];
    const bool isE = (sg & 1) == 0;
    const int64_t n = pd.n_h;
    const int64_t tile_items = kSThreads * kSelItems;
    const int64_t ntiles = (n + tile_items - 1) / tile_items;
    const int tile = claim_tile(sc.tilectr + sg, &tslot);
    if (tile < ntiles) {
        const int64_t i0 = (int64_t)tile * tile_items + (int64_t)threadIdx.x * kSelItems;
        unsigned flags = 0;
        long long cnt = 0;
        for (int i = 0; i < kSelItems; ++i) {
            const int64_t x = i0 + i;
            bool pf = false;
            if (x < n) {
                // E in halo (= id) order; R in the static (deg_in desc, id asc) order: x = rank_deg of h
                const int64_t h = isE ? x : pd.deg_order[x];
                const int32_t s = pd.slot_of[h];
                if (isE && s >= 0 && decay) {            // the same RN products as k_decay
                    const unsigned long long mask = pd.hitmask[s];
                    const int unused = decay_steps - __popcll(mask);
                    float v = pd.se[s];
                    for (int k = 0; k < unused; ++k) v = __fmul_rn(v, gamma);
                    pd.se[s] = v;
                    if (mask) pd.hitmask[s] = 0ull;
                }
                pf = isE ? (s >= 0 && pd.se[s] < alpha) : (s < 0 && pd.sa[h] >= theta_r);
            }
            flags |= (unsigned)pf << i;
            cnt += pf;
        }
        long long agg;
        long long excl = block_excl_scan256(cnt, sm, &agg);
        if (threadIdx.x < 32) {
            const unsigned long long pv = lookback_exclusive(sc.status + (int64_t)sg * tiles_max, tile,
                                                                         (unsigned long long)agg);
            if (threadIdx.x == 0) prefix_sh = (long long)pv;
        }
        __syncthreads();
        int64_t pos = prefix_sh + excl;
        const SortSeg out = segs[sg];
        uint32_t* hist = ev.hist + (size_t)sg * kDig;
        for (int i = 0; i < kSelItems; ++i) {
            const int64_t x = i0 + i;
            unsigned d = 0xFFFFFFFFu;
            if ((flags >> i) & 1u) {
                unsigned long long key;
                uint32_t val;
                if (isE) {
                    val = (uint32_t)pd.slot_of[x];
                    key = ((unsigned long long)__float_as_uint(pd.se[val]) << 32) | (uint32_t)pd.halo_ids[x];
                } else {
                    const int32_t h = pd.deg_order[x];
                    val = (uint32_t)h;
                    key = ((unsigned long long)(~__float_as_uint(pd.sa[h])) << 32) | (uint32_t)x;   // rank_deg[h] = x
                }
                MGNN_CHECK(pos < (isE ? pd.cap : n), "select pos=%lld n=%lld sg=%d", (long long)pos, (long long)n, sg);
                out.keys[pos] = key;
                out.vals[pos] = val;
                ++pos;
                d = (unsigned)(key >> 52);
            }
            const unsigned peers = __match_any_sync(kFull, d);
            if (d != 0xFFFFFFFFu && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[d], (unsigned)__popc(peers));
        }
        if (tile == ntiles - 1 && threadIdx.x == 0) n_out[sg] = prefix_sh + agg;
    } else if (ntiles == 0 && tile == 0 && threadIdx.x == 0) {
        n_out[sg] = 0;
    }
}

void launch_select(const PartDev* parts, int n_lp, int64_t n_max, float alpha, float theta_r, const SortSeg* segs,
                   long long* n_out, Scratch sc, EvScratch ev, cudaStream_t s, int decay_steps, float gamma,
                   const unsigned long long* ovf, uint64_t t_last) {
    int64_t tiles = (n_max + kSThreads * kSelItems - 1) / (kSThreads * kSelItems);
    if (tiles < 1) tiles = 1;
    dim3 grid((unsigned)tiles, 2 * n_lp);
    launch_k(k_select, grid, dim3(kSThreads), 0, s, parts, alpha, theta_r, segs, n_out, sc, tiles, ev, decay_steps,
             gamma, ovf, t_last);
    count_launches(1, __func__, s);
}

// ------------------------------------------------------------------ unordered scan (default paths)
// The K winners of each list are found from histograms and a threshold, then ranked or sorted, so
// the lists themselves never need to exist in order: k_ev_count computes |E|, |R| and the top-12-bit
// histograms straight from the scoreboards (E over the slots: S_E coalesced, the node id loaded only
// for keys that count; R over the halo), and k_ev_hist2 / k_ev_cand re-derive the same unique keys.
// Saves k_select's order-preserving compaction (look-back chain + the lists' writes).
__device__ __forceinline__ bool ev_key(const PartDev& pd, bool isE, int64_t x, float alpha, float theta_r,
                                       unsigned long long& key, uint32_t& val) {
    if (isE) {                                   // x = slot
        const float se = pd.se[x];
        if (!(se < alpha)) return false;
        const int32_t h = pd.slot_h[x];
        key = ((unsigned long long)__float_as_uint(se) << 32) | (uint32_t)pd.halo_ids[h];
        val = (uint32_t)x;
        return true;
    }
    if (pd.slot_of[x] >= 0) return false;        // x = halo index
    const float sa = pd.sa[x];
    if (!(sa >= theta_r)) return false;
    key = ((unsigned long long)(~__float_as_uint(sa)) << 32) | (uint32_t)pd.rank_deg[x];
    val = (uint32_t)x;
    return true;
}

__global__ void __launch_bounds__(kSThreads) k_ev_count(const PartDev* __restrict__ parts, float alpha, float theta_r,
                                                        long long* __restrict__ n_out, EvScratch ev) {
    pdl_enter();
    __shared__ unsigned long long cnt_sh;
    const int sg = blockIdx.y;
    const PartDev& pd = parts[sg >> 1];
    const bool isE = (sg & 1) == 0;
    const int64_t n = isE ? pd.cap : pd.n_h;
    if (threadIdx.x == 0) cnt_sh = 0;
    __syncthreads();
    uint32_t* hist = ev.hist + (size_t)sg * kDig;
    const int lane = threadIdx.x & 31;
    unsigned mine = 0;
    for (int64_t x0 = (int64_t)blockIdx.x * kSThreads; x0 < n; x0 += (int64_t)gridDim.x * kSThreads) {
        const int64_t x = x0 + threadIdx.x;
        unsigned d = 0xFFFFFFFFu;
        if (x < n) {
            bool c;
            unsigned long long key = 0;
            if (isE) {                           // the digit needs only S_E (no id load)
                const float se = pd.se[x];
                c = se < alpha;
                key = (unsigned long long)__float_as_uint(se) << 32;
            } else {
                uint32_t v;
                c = ev_key(pd, false, x, alpha, theta_r, key, v);
            }
            if (c) {
                d = (unsigned)(key >> 52);
                ++mine;
            }
        }
        const unsigned peers = __match_any_sync(kFull, d);
        if (d != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[d], (unsigned)__popc(peers));
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(kFull, mine, o);
    if (lane == 0 && mine) atomicAdd(&cnt_sh, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0 && cnt_sh) atomicAdd((unsigned long long*)&n_out[sg], cnt_sh);
}

// ------------------------------------------------------------------ candidates
// Smallest digit T with #(digit <= T) >= need (T = -1 if need <= 0); *below = #(digit < T).
// Block-wide (256 threads, 16 digits each); every block of the launch derives the same answer.
__device__ __forceinline__ void find_threshold(const uint32_t* __restrict__ hist, long long need, long long* sm,
                                               long long* T_sh, long long* below_sh) {
    constexpr int per = kDig / kSThreads;
    long long local = 0;
    for (int j = 0; j < per; ++j) local += hist[threadIdx.x * per + j];
    long long tot;
    long long run = block_excl_scan256(local, sm, &tot);
    if (threadIdx.x == 0) {
        *T_sh = -1;
        *below_sh = 0;
    }
    __syncthreads();
    if (need > 0 && run < need && need <= run + local) {
        for (int j = 0; j < per; ++j) {
            const long long c = hist[threadIdx.x * per + j];
            if (run + c >= need) {
                *T_sh = threadIdx.x * per + j;
                *below_sh = run;
                break;
            }
            run += c;
        }
    }
    __syncthreads();
}

constexpr long long kCandMax = 4096;   // refine the threshold with the next 12 key bits above this

// Second-level histogram (key bits [40, 52)) of the threshold bucket, only when the first level
// would leave more than kCandMax candidates (e.g. many equal scores in an early round).
__global__ void __launch_bounds__(kSThreads) k_hist2(const SortSeg* __restrict__ segs, EvScratch ev,
                                                     const PartDev* __restrict__ parts, float alpha, float theta_r) {
    pdl_enter();
    __shared__ long long sm[8];
    __shared__ long long T_sh, below_sh;
    const int sg = blockIdx.y;
    const SortSeg S = segs[sg];
    // parts != nullptr: the lists were never compacted; scan the scoreboards (E: slots, R: halo)
    const PartDev* pd = parts ? parts + (sg >> 1) : nullptr;
    const long long n = pd ? ((sg & 1) ? pd->n_h : pd->cap) : *S.n;
    const long long nE = *segs[sg & ~1].n, nR = *segs[sg | 1].n;
    const long long K = nE < nR ? nE : nR;
    const uint32_t* hist = ev.hist + (size_t)sg * kDig;
    find_threshold(hist, K, sm, &T_sh, &below_sh);
    const long long T = T_sh;
    if (T < 0 || below_sh + (long long)hist[T] <= kCandMax) return;
    uint32_t* hist2 = ev.hist2 + (size_t)sg * kDig;
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * kSThreads;
    for (long long i0 = (long long)blockIdx.x * kSThreads + (threadIdx.x & ~31); i0 < n; i0 += stride) {
        const long long i = i0 + lane;
        unsigned d = 0xFFFFFFFFu;
        if (i < n) {
            unsigned long long k = 0;
            uint32_t v;
            const bool c = pd ? ev_key(*pd, (sg & 1) == 0, i, alpha, theta_r, k, v) : (k = S.keys[i], true);
            if (c && (long long)(k >> 52) == T) d = (unsigned)(k >> 40) & 0xFFFu;
        }
        const unsigned peers = __match_any_sync(kFull, d);
        if (d != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist2[d], (unsigned)__popc(peers));
    }
}

// Ties beyond the two histogram levels: when the threshold bucket (the 24 key bits the histograms
// see) still holds more than kCandMax keys beyond the K needed -- e.g. thousands of R nodes with the
// same integer S_A at the threshold -- one block per list finds the exact K-th smallest key with four
// more digit passes over the low 40 bits ([28,40), [16,28), [4,16), [0,4)); k_cand then keeps exactly
// the K winners and k_rank's counting stays O(K^2).  Exits at once otherwise (one launch per round).
// Rank path only (buffers <= kEvMax slots): the sort path is linear in its candidates.
__global__ void __launch_bounds__(kSThreads) k_tie(const SortSeg* __restrict__ segs, EvScratch ev,
                                                   const PartDev* __restrict__ parts, float alpha, float theta_r) {
    pdl_enter();
    __shared__ long long sm[8];
    __shared__ long long T_sh, below_sh;
    __shared__ uint32_t h[kDig];
    const int sg = blockIdx.y;
    const SortSeg S = segs[sg];
    const PartDev* pd = parts ? parts + (sg >> 1) : nullptr;
    const long long n = pd ? ((sg & 1) ? pd->n_h : pd->cap) : *S.n;
    const long long nE = *segs[sg & ~1].n, nR = *segs[sg | 1].n;
    const long long K = nE < nR ? nE : nR;
    const uint32_t* hist = ev.hist + (size_t)sg * kDig;
    find_threshold(hist, K, sm, &T_sh, &below_sh);
    const long long T = T_sh;
    long long below = below_sh;
    if (T < 0 || below + (long long)hist[T] <= kCandMax) return;           // one level suffices
    const uint32_t* hist2 = ev.hist2 + (size_t)sg * kDig;
    find_threshold(hist2, K - below, sm, &T_sh, &below_sh);
    const long long T2 = T_sh;
    below += below_sh;
    if (below + (long long)hist2[T2] - K <= kCandMax) return;              // two levels suffice
    unsigned long long prefix = ((unsigned long long)T << 52) | ((unsigned long long)T2 << 40);
    long long need = K - below;                                            // rank inside the bucket
    const int lo_of[4] = {28, 16, 4, 0}, hi_of[4] = {40, 28, 16, 4};
    for (int lv = 0; lv < 4; ++lv) {
        const int lo = lo_of[lv], hi = hi_of[lv];
        const unsigned mask = (1u << (hi - lo)) - 1u;
        for (int d = threadIdx.x; d < kDig; d += kSThreads) h[d] = 0;
        __syncthreads();
        for (long long i = threadIdx.x; i < n; i += kSThreads) {
            unsigned long long k = 0;
            uint32_t v;
            const bool c = pd ? ev_key(*pd, (sg & 1) == 0, i, alpha, theta_r, k, v) : (k = S.keys[i], true);
            if (c && (k >> hi) == (prefix >> hi)) atomicAdd(&h[(unsigned)(k >> lo) & mask], 1u);
        }
        __syncthreads();
        find_threshold(h, need, sm, &T_sh, &below_sh);
        MGNN_CHECK(T_sh >= 0, "tie level %d: no threshold (need %lld)", lv, need);
        prefix |= (unsigned long long)T_sh << lo;
        need -= below_sh;
        __syncthreads();
    }
    if (threadIdx.x == 0) {                      // keys are unique: exactly K keys are <= prefix
        ev.kth[2 * sg] = 1ull;
        ev.kth[2 * sg + 1] = prefix;
    }
}

// Every block derives K = min(|E|, |R|) of its partition and the threshold(s) of its list from the
// histograms; block 0 records {K, T} for k_rank.
__global__ void __launch_bounds__(kSThreads) k_cand(const SortSeg* __restrict__ segs, EvScratch ev,
                                                    const PartDev* __restrict__ parts, float alpha, float theta_r) {
    pdl_enter();
    __shared__ long long sm[8];
    __shared__ long long T_sh, below_sh, T2_sh, below2_sh;
    const int sg = blockIdx.y;
    const SortSeg S = segs[sg];
    const PartDev* pd = parts ? parts + (sg >> 1) : nullptr;      // see k_hist2
    const long long n = pd ? ((sg & 1) ? pd->n_h : pd->cap) : *S.n;
    const long long nE = *segs[sg & ~1].n, nR = *segs[sg | 1].n;
    const long long K = nE < nR ? nE : nR;
    const uint32_t* hist = ev.hist + (size_t)sg * kDig;
    find_threshold(hist, K, sm, &T_sh, &below_sh);
    const long long T = T_sh;
    const bool refined = T >= 0 && below_sh + (long long)hist[T] > kCandMax;
    long long T2 = 0xFFF;
    if (refined) {
        find_threshold(ev.hist2 + (size_t)sg * kDig, K - below_sh, sm, &T2_sh, &below2_sh);
        T2 = T2_sh;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ev.thr[2 * sg] = K;
        ev.thr[2 * sg + 1] = T;
    }
    if (T < 0) return;
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * kSThreads;
    const bool exact = ev.kth[2 * sg] != 0ull;   // k_tie resolved the K-th key exactly
    const unsigned long long kth = ev.kth[2 * sg + 1];
    for (long long i0 = (long long)blockIdx.x * kSThreads + (threadIdx.x & ~31); i0 < n; i0 += stride) {
        const long long i = i0 + lane;
        unsigned long long k = 0;
        uint32_t v = 0;
        bool c = false;
        if (i < n) {
            const bool in = pd ? ev_key(*pd, (sg & 1) == 0, i, alpha, theta_r, k, v) : (k = S.keys[i], v = S.vals[i], true);
            const long long d1 = (long long)(k >> 52);
            c = in && (exact ? k <= kth : (d1 < T || (d1 == T && (long long)((k >> 40) & 0xFFF) <= T2)));
        }
        const unsigned ball = __ballot_sync(kFull, c);
        if (!ball) continue;
        // warp-aggregated append (order irrelevant: keys are unique)
        unsigned long long base = 0;
        const int leader = __ffs(ball) - 1;
        if (lane == leader) base = atomicAdd(&ev.n_cand[sg], (unsigned long long)__popc(ball));
        base = __shfl_sync(kFull, base, leader);
        if (c) {
            const unsigned long long p = base + __popc(ball & ((1u << lane) - 1u));
            S.keys_tmp[p] = k;
            S.vals_tmp[p] = v;
        }
    }
}

// Order-preserving variant for the compacted lists (k_select): tiles of 2048 list entries claimed in
// order, block scan + decoupled look-back, so the candidates keep the list order -- E by id, R by
// rank_deg, i.e. the order of each key's low word -- and the K winners need a stable sort of the HIGH
// word only (4 digit passes instead of 8).  Same thresholds as k_cand.
__global__ void __launch_bounds__(kSThreads) k_cand_ord(const SortSeg* __restrict__ segs, EvScratch ev, Scratch sc,
                                                        int64_t tiles_max) {
    pdl_enter();
    __shared__ long long sm[8];
    __shared__ long long T_sh, below_sh, T2_sh, below2_sh, prefix_sh;
    __shared__ int tslot;
    const int sg = blockIdx.y;
    const SortSeg S = segs[sg];
    const long long n = *S.n;
    const long long nE = *segs[sg & ~1].n, nR = *segs[sg | 1].n;
    const long long K = nE < nR ? nE : nR;
    const uint32_t* hist = ev.hist + (size_t)sg * kDig;
    find_threshold(hist, K, sm, &T_sh, &below_sh);
    const long long T = T_sh;
    const bool refined = T >= 0 && below_sh + (long long)hist[T] > kCandMax;
    long long T2 = 0xFFF;
    if (refined) {
        find_threshold(ev.hist2 + (size_t)sg * kDig, K - below_sh, sm, &T2_sh, &below2_sh);
        T2 = T2_sh;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ev.thr[2 * sg] = K;
        ev.thr[2 * sg + 1] = T;
    }
    if (T < 0) return;                           // same answer in every block of the segment
    const int64_t tile_items = kSThreads * kSelItems;
    const int64_t ntiles = (n + tile_items - 1) / tile_items;
    const int tile = claim_tile(sc.tilectr + sg, &tslot);
    if (tile >= ntiles) return;
    const int64_t i0 = (int64_t)tile * tile_items + (int64_t)threadIdx.x * kSelItems;
    unsigned long long k[kSelItems];
    unsigned flags = 0;
    long long cnt = 0;
#pragma unroll
    for (int i = 0; i < kSelItems; ++i) {
        k[i] = i0 + i < n ? S.keys[i0 + i] : ~0ull;
        const long long d1 = (long long)(k[i] >> 52);
        const bool c = i0 + i < n && (d1 < T || (d1 == T && (long long)((k[i] >> 40) & 0xFFF) <= T2));
        flags |= (unsigned)c << i;
        cnt += c;
    }
    long long agg;
    const long long excl = block_excl_scan256(cnt, sm, &agg);
    if (threadIdx.x < 32) {
        const unsigned long long pv = lookback_exclusive(sc.status + (int64_t)sg * tiles_max, tile,
                                                         (unsigned long long)agg);
        if (threadIdx.x == 0) prefix_sh = (long long)pv;
    }
    __syncthreads();
    long long pos = prefix_sh + excl;
#pragma unroll
    for (int i = 0; i < kSelItems; ++i)
        if ((flags >> i) & 1u) {
            S.keys_tmp[pos] = k[i];
            S.vals_tmp[pos] = S.vals[i0 + i];
            ++pos;
        }
    if (tile == ntiles - 1 && threadIdx.x == 0) ev.n_cand[sg] = (unsigned long long)(prefix_sh + agg);
}

// ------------------------------------------------------------------ rank by counting (unique keys)
__global__ void __launch_bounds__(kSThreads) k_rank(const SortSeg* __restrict__ segs, EvScratch ev) {
    pdl_enter();
    __shared__ unsigned long long tile_k[2048];
    const int sg = blockIdx.y;
    const SortSeg S = segs[sg];
    const long long T = ev.thr[2 * sg + 1];
    if (T < 0) return;
    const long long nc = (long long)ev.n_cand[sg];
    const long long K = ev.thr[2 * sg];
    const long long first = (long long)blockIdx.x * kSThreads;
    if (first >= nc) return;
    const long long c = first + threadIdx.x;
    const unsigned long long mine = c < nc ? S.keys_tmp[c] : ~0ull;
    long long rank = 0;
    for (long long t0 = 0; t0 < nc; t0 += 2048) {
        const int m = (int)(nc - t0 < 2048 ? nc - t0 : 2048);
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += kSThreads) tile_k[j] = S.keys_tmp[t0 + j];
        __syncthreads();
        int r = 0;
#pragma unroll 8
        for (int j = 0; j < m; ++j) r += tile_k[j] < mine;
        rank += r;
    }
    if (c < nc && rank < K) {
        S.keys[rank] = mine;          // the K winners, in order, replace the list
        S.vals[rank] = S.vals_tmp[c];
    }
}

void launch_ev_count(const PartDev* parts, int n_lp, int64_t n_max, float alpha, float theta_r, long long* n_out,
                     EvScratch ev, cudaStream_t s) {
    dim3 grid(blocks_for(n_max, kSThreads), 2 * n_lp);
    launch_k(k_ev_count, grid, dim3(kSThreads), 0, s, parts, alpha, theta_r, n_out, ev);
    count_launches(1, __func__, s);
}

void launch_cand(const SortSeg* segs, int n_lp, int64_t n_max, EvScratch ev, const PartDev* scan_parts, float alpha,
                 float theta_r, cudaStream_t s) {
    const unsigned cap_blocks = scan_parts ? 256u : 64u;     // the scoreboard scan covers all of n_h
    dim3 g1(blocks_for(n_max, kSThreads) > cap_blocks ? cap_blocks : blocks_for(n_max, kSThreads), 2 * n_lp);
    // (no k_tie here: the radix sort is linear in the candidates, ties only cost their sort passes)
    launch_k(k_hist2, g1, dim3(kSThreads), 0, s, segs, ev, scan_parts, alpha, theta_r);
    launch_k(k_cand, g1, dim3(kSThreads), 0, s, segs, ev, scan_parts, alpha, theta_r);
    count_launches(2, __func__, s);
}

void launch_cand_ord(const SortSeg* segs, int n_lp, int64_t n_max, EvScratch ev, Scratch sc, int64_t tiles_max,
                     cudaStream_t s) {
    const unsigned cap_blocks = 64u;
    dim3 g1(blocks_for(n_max, kSThreads) > cap_blocks ? cap_blocks : blocks_for(n_max, kSThreads), 2 * n_lp);
    launch_k(k_hist2, g1, dim3(kSThreads), 0, s, segs, ev, (const PartDev*)nullptr, 0.0f, 0.0f);
    int64_t tiles = (n_max + kSThreads * kSelItems - 1) / (kSThreads * kSelItems);
    if (tiles < 1) tiles = 1;
    launch_k(k_cand_ord, dim3((unsigned)tiles, 2 * n_lp), dim3(kSThreads), 0, s, segs, ev, sc, tiles_max);
    count_launches(2, __func__, s);
}

void launch_cand_rank(const SortSeg* segs, int n_lp, int64_t n_max, EvScratch ev, const PartDev* scan_parts,
                      float alpha, float theta_r, cudaStream_t s) {
    const unsigned cap_blocks = scan_parts ? 256u : 64u;
    dim3 g1(blocks_for(n_max, kSThreads) > cap_blocks ? cap_blocks : blocks_for(n_max, kSThreads), 2 * n_lp);
    launch_k(k_hist2, g1, dim3(kSThreads), 0, s, segs, ev, scan_parts, alpha, theta_r);
    launch_k(k_tie, dim3(1, 2 * n_lp), dim3(kSThreads), 0, s, segs, ev, scan_parts, alpha, theta_r);
    launch_k(k_cand, g1, dim3(kSThreads), 0, s, segs, ev, scan_parts, alpha, theta_r);
    dim3 g2((unsigned)((n_max + kSThreads - 1) / kSThreads), 2 * n_lp);
    launch_k(k_rank, g2, dim3(kSThreads), 0, s, segs, ev);
    count_launches(4, __func__, s);
}

// ------------------------------------------------------------------ swap + refill
// Pair i (i < k = min(|E|, |R|), R#19): slot s = E[i], evicted e, replacement r = R[i]:
//   S_A[e] <- S_E[s]; slot_of[e] <- -1; BUF[s] <- r; S_E[s] <- S_A[r]; S_A[r] <- -1
// then the row of r is copied from its owner's table into the slot.
// E and R are disjoint (buffered vs. not), so pairs never conflict.
__global__ void __launch_bounds__(kSThreads) k_swap_refill(const PartDev* __restrict__ parts,
                                                           const SortSeg* __restrict__ segs,
                                                           const long long* __restrict__ k_of, WorldDev G,
                                                           long long* counts, int64_t counts_stride, int n_steps,
                                                           const unsigned long long* ovf, uint64_t t_last) {
    pdl_enter();
    if (*ovf <= t_last) return;                  // arena overflow: the window was skipped
    const int lp = blockIdx.y;
    const PartDev& pd = parts[lp];
    const SortSeg E = segs[2 * lp], R = segs[2 * lp + 1];
    const long long nE = *E.n, nR = *R.n;
    const long long k = k_of ? k_of[4 * lp] : (nE < nR ? nE : nR);   // k_of: {K, T} per segment
    const int lane = threadIdx.x & 31;
    const int pitch = G.pitch;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        long long* cn = counts + ((int64_t)lp * n_steps + (n_steps - 1)) * counts_stride;
        cn[4] = k;
        cn[5] = k;
        cn[6] += k;
    }
    const int64_t nwarps = (int64_t)gridDim.x * (kSThreads / 32);
    for (int64_t i = (int64_t)blockIdx.x * (kSThreads / 32) + (threadIdx.x >> 5); i < k; i += nwarps) {
        const int32_t s = (int32_t)E.vals[i];
        const int32_t r = (int32_t)R.vals[i];
        MGNN_CHECK(s >= 0 && s < pd.cap && r >= 0 && r < pd.n_h, "swap lp=%d i=%lld s=%d r=%d", lp, (long long)i, s,
                   r);
        if (lane == 0) {
            const int32_t e = pd.slot_h[s];
            const float se_s = pd.se[s];
            const float sa_r = pd.sa[r];
            pd.sa[e] = se_s;
            pd.slot_of[e] = -1;
            pd.slot_h[s] = r;
            pd.slot_of[r] = s;
            pd.se[s] = sa_r;
            pd.sa[r] = -1.0f;
        }
        const int32_t gid = pd.halo_ids[r];
        const int q = owner_of(G.bounds, G.n_parts, gid);
        const float* src = G.tables[q] + ((int64_t)gid - G.bounds[q]) * pitch;
        float* dst = pd.rows + (int64_t)s * pitch;
        for (int c = lane * 4; c < pitch; c += 128)
            *reinterpret_cast<float4*>(dst + c) = __ldg(reinterpret_cast<const float4*>(src + c));
        if (lane == 0 && G.on_peer[q])
            atomicAdd((unsigned long long*)(counts + ((int64_t)lp * n_steps + (n_steps - 1)) * counts_stride + 7), 1ull);
    }
}

void launch_swap_refill(const PartDev* parts, int n_lp, int64_t cap_max, const SortSeg* segs, const long long* k_of,
                        const WorldDev& world,
                        long long* counts, int64_t counts_stride, int n_steps, const unsigned long long* ovf,
                        uint64_t t_last, cudaStream_t s) {
    dim3 grid(blocks_for(cap_max < 1 ? 1 : cap_max, kSThreads / 32), n_lp);
    launch_k(k_swap_refill, grid, dim3(kSThreads), 0, s, parts, segs, k_of, world, counts, counts_stride, n_steps,
             ovf, t_last);
    count_launches(1, __func__, s);
}

// ------------------------------------------------------------------ INITIALIZE_PREFETCHER
// keys = ~deg_in (ascending = degree desc), values = halo index in id order.
__global__ void k_init_keys(const PartDev* __restrict__ pdp, const SortSeg* __restrict__ seg, long long* n_dev) {
    const PartDev& pd = *pdp;
    const SortSeg sg = *seg;
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < pd.n_h; h += (int64_t)gridDim.x * blockDim.x) {
        sg.keys[h] = (unsigned long long)(~(uint32_t)pd.deg_in[h]);
        sg.vals[h] = (uint32_t)h;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = pd.n_h;
}

void launch_init_keys(const PartDev* pd_dev, int64_t n_h, const SortSeg* seg, long long* n_dev, cudaStream_t s) {
    k_init_keys<<<blocks_for(n_h < 1 ? 1 : n_h, kSThreads), kSThreads, 0, s>>>(pd_dev, seg, n_dev);
    count_launches(1, __func__, s);
}

// S_A = 0 for every halo node and rank_deg[order[i]] = i; then for the top-cap: slot s <- order[s],
// S_E = 1, S_A = -1.
__global__ void k_init_reset(const PartDev* __restrict__ pdp, const uint32_t* __restrict__ order) {
    const PartDev& pd = *pdp;
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < pd.n_h; h += (int64_t)gridDim.x * blockDim.x) {
        pd.sa[h] = 0.0f;
        pd.slot_of[h] = -1;
        pd.rank_deg[order[h]] = (int32_t)h;
        pd.deg_order[h] = (int32_t)order[h];
    }
}

__global__ void k_init_slots(const PartDev* __restrict__ pdp, const uint32_t* __restrict__ order) {
    const PartDev& pd = *pdp;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < pd.cap; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t h = (int32_t)order[s];
        pd.slot_h[s] = h;
        pd.slot_of[h] = (int32_t)s;
        pd.se[s] = 1.0f;
        pd.sa[h] = -1.0f;
        pd.hitmask[s] = 0ull;
    }
}

void launch_init_fill(const PartDev* pd_dev, int64_t n_h, int64_t cap, const uint32_t* order, cudaStream_t s) {
    k_init_reset<<<blocks_for(n_h < 1 ? 1 : n_h, kSThreads), kSThreads, 0, s>>>(pd_dev, order);
    k_init_slots<<<blocks_for(cap < 1 ? 1 : cap, kSThreads), kSThreads, 0, s>>>(pd_dev, order);
    count_launches(2, __func__, s);
}

// BUF rows of every slot from the owners' tables (the init "RPC").
__global__ void k_rows_from_owners(const PartDev* __restrict__ pdp, WorldDev G) {
    const PartDev& pd = *pdp;
    const int lane = threadIdx.x & 31;
    const int pitch = G.pitch;
    for (int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); s < pd.cap;
         s += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int32_t gid = pd.halo_ids[pd.slot_h[s]];
        const int q = owner_of(G.bounds, G.n_parts, gid);
        const float* src = G.tables[q] + ((int64_t)gid - G.bounds[q]) * pitch;
        float* dst = pd.rows + s * pitch;
        for (int c = lane * 4; c < pitch; c += 128)
            *reinterpret_cast<float4*>(dst + c) = __ldg(reinterpret_cast<const float4*>(src + c));
    }
}

void launch_rows_from_owners(const PartDev* pd_dev, int64_t cap, const WorldDev& world, cudaStream_t s) {
    if (cap < 1) return;
    k_rows_from_owners<<<blocks_for(cap, kSThreads / 32), kSThreads, 0, s>>>(pd_dev, world);
    count_launches(1, __func__, s);
}

// ------------------------------------------------------------------ epoch orders (R#8)
// G epoch orders of a partition at once: train ids sorted by (Philox key, id).  MSB bucket
// scheme instead of an LSD sort: (1) keys + histogram of the top key byte, (2) scatter into the
// 256 buckets of each epoch, (3) one block per bucket ranks its items by counting smaller
// (key, index) pairs -- the rank is the sorted position.  Philox keys are uniform, so a bucket
// holds ~n/256 items; any size stays correct (large buckets are ranked from global memory).
__global__ void k_perm_keys(const PartDev* __restrict__ pdp, uint64_t epoch0, int n_epochs, uint32_t k0, uint32_t k1,
                            const SortSeg* __restrict__ segs, uint32_t* __restrict__ hist) {
    const PartDev& pd = *pdp;
    const uint32_t c3 = ((uint32_t)pd.part_id << 8) | kStreamShuffle;
    const int64_t n = pd.n_train, total = n * n_epochs;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = x / n, i = x - j * n;
        const uint32_t id = (uint32_t)pd.train_ids[i];
        const u4 o = philox4x32_10(u4{id, (uint32_t)(epoch0 + j), 0u, c3}, k0, k1);
        const unsigned long long key = ((unsigned long long)o.x << 32) | o.y;
        segs[j].keys[i] = key;
        atomicAdd(&hist[j * 256 + (unsigned)(key >> 56)], 1u);
    }
}

// exclusive prefix of the segment's 256 bucket counts, in shared memory (256 threads)
__device__ __forceinline__ void bucket_starts(const uint32_t* __restrict__ h, uint32_t* start_sh, long long* sm) {
    long long tot;
    const long long ex = block_excl_scan256(h[threadIdx.x], sm, &tot);
    start_sh[threadIdx.x] = (uint32_t)ex;
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_perm_scatter(const PartDev* __restrict__ pdp, int n_epochs,
                                                      const SortSeg* __restrict__ segs, const uint32_t* __restrict__ hist,
                                                      uint32_t* __restrict__ cursor) {
    pdl_enter();
    __shared__ uint32_t start[256];
    __shared__ long long sm[8];
    const int64_t n = pdp->n_train;
    const int j = blockIdx.y;
    bucket_starts(hist + j * 256, start, sm);
    const SortSeg sg = segs[j];
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
        const unsigned long long key = sg.keys[i];
        const unsigned b = (unsigned)(key >> 56);
        const uint32_t p = start[b] + atomicAdd(&cursor[j * 256 + b], 1u);
        sg.keys_tmp[p] = key;
        sg.vals_tmp[p] = (uint32_t)i;         // list index = id order: the tie-break
    }
}

__global__ void __launch_bounds__(256) k_perm_rank(const PartDev* __restrict__ pdp, const SortSeg* __restrict__ segs,
                                                   const uint32_t* __restrict__ hist) {
    pdl_enter();
    __shared__ uint32_t start[256];
    __shared__ long long sm[8];
    __shared__ unsigned long long sk[1024];
    __shared__ uint32_t si[1024];
    const int j = blockIdx.y, b = blockIdx.x;
    bucket_starts(hist + j * 256, start, sm);
    const SortSeg sg = segs[j];
    const uint32_t s0 = start[b], cnt = hist[j * 256 + b];
    const bool in_smem = cnt <= 1024;
    if (in_smem) {
        for (uint32_t x = threadIdx.x; x < cnt; x += 256) {
            sk[x] = sg.keys_tmp[s0 + x];
            si[x] = sg.vals_tmp[s0 + x];
        }
        __syncthreads();
    }
    const int32_t* train = pdp->train_ids;
    for (uint32_t x = threadIdx.x; x < cnt; x += 256) {
        const unsigned long long k = in_smem ? sk[x] : sg.keys_tmp[s0 + x];
        const uint32_t i = in_smem ? si[x] : sg.vals_tmp[s0 + x];
        uint32_t rank = 0;
        for (uint32_t y = 0; y < cnt; ++y) {
            const unsigned long long ky = in_smem ? sk[y] : sg.keys_tmp[s0 + y];
            const uint32_t iy = in_smem ? si[y] : sg.vals_tmp[s0 + y];
            rank += (ky < k) || (ky == k && iy < i);
        }
        sg.vals[s0 + rank] = (uint32_t)train[i];   // vals = the epoch-order slot
    }
}

void launch_perm_build(const PartDev* pd_dev, int64_t n_train, uint64_t epoch0, int n_epochs, uint32_t seed_lo,
                       uint32_t seed_hi, const SortSeg* segs, void* scratch, cudaStream_t s) {
    uint32_t* hist = (uint32_t*)scratch;
    uint32_t* cursor = hist + (size_t)n_epochs * 256;
    cudaMemsetAsync(scratch, 0, (size_t)n_epochs * 256 * 2 * sizeof(uint32_t), s);
    const int64_t total = n_train * n_epochs;
    k_perm_keys<<<blocks_for(total < 1 ? 1 : total, kSThreads), kSThreads, 0, s>>>(pd_dev, epoch0, n_epochs, seed_lo,
                                                                                   seed_hi, segs, hist);
    unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_train + 255) / 256, 64));
    launch_k(k_perm_scatter, dim3(gx, n_epochs), dim3(256), 0, s, pd_dev, n_epochs, segs, (const uint32_t*)hist, cursor);
    launch_k(k_perm_rank, dim3(256, n_epochs), dim3(256), 0, s, pd_dev, segs, (const uint32_t*)hist);
    count_launches(3, __func__, s);
}

}  // namespace mgnn
