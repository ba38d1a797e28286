// sample.cu -- NeighborSampler of Alg.2 l.1 (uniform fixed
// fanout without replacement) for a window of minibatch instances.
//
// Work unit: instance m = (local partition lp, window step w).  All kernels
// run every instance of the window side by side (gridDim.y = instances), so
// one launch per stage serves W steps x P_local partitions.
//
// Per hop i (K1/K2):
//   k_hop     : thread per frontier node x of F_i (a tile of 256 per block):
//               count min(deg, k_i) (halo nodes: 0, R#1), exclusive offsets by
//               a block scan + decoupled look-back across tiles; then groups
//               of G = pow2 >= k_i lanes take the tile's nodes 32/G per warp
//               at a time: lane j draws u_j = Philox(x, (i<<16)|j, step,
//               (p<<8)|1) (R#4), r_j = mulhi(u_j, t_j+1) (R#5), Floyd
//               resolution by k_i in-group shuffles (R#6), and stages the
//               CSR index in shared memory; finally all threads of the block
//               load the neighbours' local ranks in parallel, write them in
//               slot order (coalesced) and mark them in the new-node bitmap
//               unless already in F_i.
//   k_compact : the bitmap in rank order IS the ascending-id order, so a
//               popcount scan appends sorted_unique(cols_i) \ F_i to the
//               frontier (R#7) and keeps, beside each bitmap word, the
//               frontier position of its first new node (one 8-byte pair).
// After the last hop k_relabel rewrites the sampled columns as positions in
// F_{i+1} (the DGL block layout the consumer indexes X with): a new node's
// position is its word's position + popc of the lower bits of new_j.
#include <cstdlib>

#include "launch.h"

namespace mgnn {

constexpr int kThreads = 256;
constexpr int kHopTileMin = 64;        // frontier nodes per k_hop tile: 64 or 256
constexpr int kCWords = 4;             // bitmap words per k_compact thread (2 16-byte loads of pairs)
constexpr int kRelabelBatch = 4;       // column lookups in flight per k_relabel thread (8: no gain)
#ifndef MGNN_HOP_BLOCKS
#define MGNN_HOP_BLOCKS 8                // resident k_hop blocks per SM (32 registers; 5 x 8 loads: +11 % hop time)
#endif
#ifndef MGNN_COL_BATCH
#define MGNN_COL_BATCH 4
#endif
constexpr int kColBatch = MGNN_COL_BATCH;           // neighbour-rank loads in flight per k_hop thread
constexpr int kWordTile = kThreads * kCWords;   // bitmap words per k_compact tile
constexpr int kCompactStage = 4096;             // new ranks of a tile staged in shared memory (16 KB)

// + kMaxLayers + 1: segment-aligned tiles (k_hop align) may leave one partial tile per segment
int64_t scan_tiles_count(int64_t fcap) { return (fcap + kHopTileMin - 1) / kHopTileMin + kMaxLayers + 1; }
int64_t scan_tiles_words(int64_t words) { return (words + kWordTile - 1) / kWordTile; }

static inline unsigned grid_x_for(int64_t items_per_inst, int items_per_block, int n_inst) {
    // enough blocks to cover one instance, but about 16 resident blocks per SM overall
    int64_t need = (items_per_inst + items_per_block - 1) / items_per_block;
    int64_t target = ((int64_t)num_sms() * 16 + n_inst - 1) / n_inst;
    int64_t g = need < target ? need : target;
    return (unsigned)(g < 1 ? 1 : g);
}

__device__ __forceinline__ uint32_t seed_hash(int32_t r) { return (uint32_t)r * 0x9E3779B1u >> 7; }

// ------------------------------------------------------------------ seeds: F_0 (R#8)
__global__ void __launch_bounds__(kThreads) k_seeds(WinDev W) {
    pdl_enter();
    const int m = blockIdx.y;
    const int lp = m / W.n_steps, w = m % W.n_steps;
    const PartDev& pd = W.parts[lp];
    const uint64_t t = W.step0 + (uint64_t)w;
    const int32_t* src;
    int64_t n0;
    if (W.ext_seeds) {
        src = W.ext_seeds + (int64_t)m * W.batch;
        n0 = W.ext_counts[m];
        if (n0 < 1 || n0 > W.batch) {
            if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(W.err, 1);
            n0 = 0;
        }
    } else {
        const int64_t e = (int64_t)((t - 1) / (uint64_t)pd.nbatch), b = (int64_t)((t - 1) % (uint64_t)pd.nbatch);
        const int32_t* perm = pd.perm + (int64_t)(e % pd.perm_slots) * pd.n_train;
        const int64_t s0 = b * W.batch;
        n0 = pd.n_train - s0 < W.batch ? pd.n_train - s0 : W.batch;
        src = perm + s0;
    }
    int32_t* fr = W.fr_rank + (int64_t)m * W.ucap;
    int2* sp = W.seedpos + (int64_t)m * (W.seed_hmask + 1);
    uint32_t* fb = W.fb + (int64_t)m * W.bm_words;
    uint32_t* fbp = W.fbp + (int64_t)m * W.bm_words;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n0; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gid = src[j];
        int64_t row = gid - pd.lo;
        if (row < 0 || row >= pd.n_local) {      // external seed not owned by this partition
            atomicOr(W.err, 1);
            row = 0;
        }
        const int32_t r = (int32_t)((W.remote ? pd.lo : pd.h_below) + row);   // rank (= global id when remote)
        MGNN_CHECK(j < W.ucap, "seed position %lld", (long long)j);
        fr[j] = r;
        W.fr_gid[(int64_t)m * W.ucap + j] = (int32_t)gid;   // F_0 readable right after sampling
        for (uint32_t h = seed_hash(r) & (uint32_t)W.seed_hmask;; h = (h + 1) & (uint32_t)W.seed_hmask) {
            const int prev = atomicCAS(&sp[h].x, 0, r + 1);        // open addressing, key = rank + 1
            if (prev == 0 || prev == r + 1) {
                sp[h].y = (int32_t)j;
                break;
            }
        }
        const uint32_t bit = 1u << (r & 31);
        if (W.ext_seeds) {                                  // user seeds: detect duplicates
            if (atomicOr(&fb[r >> 5], bit) & bit) atomicOr(W.err, 2);
        } else {                                            // epoch order: distinct by construction
            atomicOr(&fb[r >> 5], bit);
        }
        atomicOr(&fbp[r >> 5], bit);                        // F_0 = the frontier before hop 0
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) W.hop_size[(int64_t)m * (kMaxLayers + 1)] = n0;
}

// ------------------------------------------------------------------ one hop: counts, offsets, samples
// T = frontier nodes per tile (64 or 256; small tiles give small hops enough blocks).
// Per tile: (1) thread per node: deg-capped count, block scan -> tile-relative
// sample offsets; (2) warp 0 resolves the tile's global offset by look-back
// while warps 1..7 produce the CSR index of every sample (a node with deg <= k
// takes its whole neighbourhood, R#3; a node with deg > k is drawn by a group
// of k lanes: Philox + Floyd, R#4-R#6); (3) all threads load the sampled
// neighbours' ranks, write the columns (coalesced) and mark new nodes.
template <typename IdxT>   // CSR index staged per sample: uint32_t when every index fits (halves the tile)
__global__ void __launch_bounds__(kThreads, MGNN_HOP_BLOCKS) k_hop(WinDev W, int hop, Scratch sc, int64_t tiles_max, int T,
                                                                     int mark_filter, int align, int one_tile) {
    pdl_enter();
    __shared__ long long sm[8];
    __shared__ int tslot, n_draw;
    __shared__ long long prefix_sh;
    __shared__ long long s_b0[kThreads];
    __shared__ int s_row[kThreads], s_d[kThreads], s_o[kThreads], s_draw[kThreads];
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    IdxT* sidx = reinterpret_cast<IdxT*>(dyn_smem);   // [T * k] CSR index of each sample of the tile
    const int m = blockIdx.y;
    const int lp = m / W.n_steps, w = m % W.n_steps;
    const PartDev& pd = W.parts[lp];
    const int64_t* hsm = W.hop_size + (int64_t)m * (kMaxLayers + 1);
    const int64_t nF = hsm[hop];
    // align != 0: segment-aligned tiles.  F_hop = F_0 ++ new_0 ++ ... ++ new_{hop-1}, each segment in rank
    // order (R#7); tile c of segment s covers the fraction [c, c+1) / C_s of that segment in EVERY
    // instance (C_s = ceil(longest segment s of the window / T)), so the instances, whose blocks claim
    // their tiles in step, sample the same rank region -- the same CSR rows -- at the same time (L2
    // reuse of rows that several minibatches of the window expand).  Tiles stay contiguous and in
    // frontier order, as the decoupled look-back requires.
    __shared__ long long seg_c[kMaxLayers + 2];
    int64_t ntiles = (nF + T - 1) / T;
    if (align) {
        if (threadIdx.x < kMaxLayers + 2) seg_c[threadIdx.x] = 0;
        __syncthreads();
        for (int mi = threadIdx.x; mi < W.n_inst; mi += blockDim.x) {
            const int64_t* hsi = W.hop_size + (int64_t)mi * (kMaxLayers + 1);
            for (int sgi = 0; sgi <= hop; ++sgi) {
                const long long len = sgi == 0 ? hsi[0] : hsi[sgi] - hsi[sgi - 1];
                atomicMax(&seg_c[sgi + 1], (len + T - 1) / T);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int sgi = 1; sgi <= hop + 1; ++sgi) seg_c[sgi] += seg_c[sgi - 1];
        __syncthreads();
        ntiles = seg_c[hop + 1];
    }
    int64_t* off = W.off[hop] + (int64_t)m * W.off_stride[hop];
    const int k = W.k_hop[hop];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = 32 / k;                                // k lanes per drawn node, `per` nodes per warp step
    const int gi = lane / k, gl = lane - gi * k, gbase = gi * k;
    const uint32_t c1 = (uint32_t)hop << 16;
    const uint32_t c3 = ((uint32_t)pd.part_id << 8) | kStreamSample;
    const uint32_t step = (uint32_t)(W.step0 + (uint64_t)w);
    const int64_t h_below = pd.h_below, n_local = pd.n_local, lo = pd.lo;
    // persistent: blocks claim tiles in order until the instance's frontier is exhausted (one_tile: a
    // block takes one tile and exits, so blocks of other streams' kernels get SM slots as it runs)
    for (int done = 0;; ++done) {
        if (one_tile && done) break;
        if (threadIdx.x == 0) n_draw = 0;
        const int tile = claim_tile(sc.tilectr + m, &tslot);
        if (tile >= ntiles) {
            if (tile == 0 && threadIdx.x == 0) off[0] = 0;   // empty F_i
            break;
        }
        int64_t f = (int64_t)tile * T + threadIdx.x, f_end = nF;
        if (align) {                                       // the tile's slice of its segment
            int sgi = 0;
            while (tile >= seg_c[sgi + 1]) ++sgi;
            const int64_t c = tile - seg_c[sgi], C = seg_c[sgi + 1] - seg_c[sgi];
            const int64_t s0 = sgi == 0 ? 0 : hsm[sgi - 1], len = sgi == 0 ? hsm[0] : hsm[sgi] - hsm[sgi - 1];
            f = s0 + c * len / C + threadIdx.x;
            f_end = s0 + (c + 1) * len / C;
        }
        const bool mine = threadIdx.x < T && f < f_end;
        int64_t row = -1, b0 = 0, d = 0;
        if (mine) {
            const int64_t r = W.fr_rank[(int64_t)m * W.ucap + f];
            if (W.remote) {                                // NEXT-1: every node, from the global CSR
                row = r - lo;                              // (rank = global id; lo + row = id)
                b0 = W.g_indptr[r];
                d = W.g_indptr[r + 1] - b0;
            } else {
                row = r - h_below;
                if (row >= 0 && row < n_local) {           // halo frontier nodes are leaves (R#1)
                    b0 = pd.indptr[row];
                    d = pd.indptr[row + 1] - b0;
                } else {
                    row = -1;
                }
            }
        }
        const int cnt = (int)(d < k ? d : k);              // |sample| = min(deg, k) (R#3)
        long long agg;
        const int excl = (int)block_excl_scan256(cnt, sm, &agg);   // tile-relative offset (< T * k)
        if (threadIdx.x < T) s_o[threadIdx.x] = excl;
        const bool draw = cnt > 0 && d > k;
        if (cnt > 0 && !draw)                              // whole neighbourhood in CSR order (R#3)
            for (int j = 0; j < cnt; ++j) sidx[excl + j] = (IdxT)(b0 + j);
        const unsigned bal = __ballot_sync(kFull, draw);
        int dbase = 0;
        if (lane == 0 && bal) dbase = atomicAdd(&n_draw, __popc(bal));
        dbase = __shfl_sync(kFull, dbase, 0);
        if (draw) {
            s_draw[dbase + __popc(bal & ((1u << lane) - 1u))] = threadIdx.x;
            s_row[threadIdx.x] = (int)row;
            s_b0[threadIdx.x] = b0;
            s_d[threadIdx.x] = (int)d;
        }
        __syncthreads();
        if (warp == 0) {
            // global offset of the tile; overlaps with the sample draws of warps 1..7
            const unsigned long long pv =
                lookback_exclusive(sc.status + (int64_t)m * tiles_max, tile, (unsigned long long)agg);
            if (lane == 0) prefix_sh = (long long)pv;
        } else {
            // drawn nodes: k lanes per node, lane j draws slot j; Floyd collisions by k in-group shuffles
            const int nd = n_draw;
            for (int bd = (warp - 1) * per; bd < nd; bd += 7 * per) {
                const int di = bd + gi;
                const bool active = gi < per && di < nd;
                const int x = active ? s_draw[di] : 0;
                uint32_t r = 0, t = 0;
                bool coll = false;
                if (active) {
                    const u4 u = philox4x32_10(u4{(uint32_t)(lo + s_row[x]), c1 | (uint32_t)gl, step, c3},
                                               W.seed_lo, W.seed_hi);
                    t = (uint32_t)(s_d[x] - k + gl);
                    r = __umulhi(u.x, t + 1u);             // floor(u (t+1) / 2^32)
                }
                for (int jj = 0; jj < k; ++jj) {           // Floyd: pos_j = r_j unless already chosen, else t_j
                    const uint32_t pj = __shfl_sync(kFull, coll ? t : r, (gbase + jj) & 31);
                    if (gl > jj && r == pj) coll = true;
                }
                if (active) sidx[s_o[x] + gl] = (IdxT)(s_b0[x] + (coll ? t : r));
            }
        }
        __syncthreads();
        // every sample of the tile in parallel: neighbour rank, coalesced column write, new-node mark
        const long long o_tile = prefix_sh;
        if (mine) {
            MGNN_CHECK(f + 1 < W.off_stride[hop], "off f=%lld", (long long)f);
            off[f + 1] = o_tile + excl + cnt;
        }
        if (tile == 0 && threadIdx.x == 0) off[0] = 0;
        int32_t* cols = W.cols[hop] + (int64_t)m * W.col_stride[hop] + o_tile;
        uint32_t* fb = W.fb + (int64_t)m * W.bm_words;
        const int32_t* __restrict__ crank = W.remote ? W.g_cols : pd.cols_rank;
        // batches of kColBatch samples per thread: all neighbour-rank loads in flight, then the column
        // writes and the membership marks: every sampled rank is OR-ed into the cumulative frontier
        // bitmap fb (a fire-and-forget reduction; k_compact finds new_i = fb & ~F_i).  mark_filter = 1
        // loads the word first and skips ranks already present.
        for (int e0 = threadIdx.x; e0 < (int)agg; e0 += kThreads * kColBatch) {
            int32_t c[kColBatch];
            uint32_t fw[kColBatch];
#pragma unroll
            for (int j = 0; j < kColBatch; ++j) {
                const int e = e0 + j * kThreads;
                c[j] = e < (int)agg ? __ldg(crank + sidx[e]) : -1;
            }
            if (mark_filter) {
#pragma unroll
                for (int j = 0; j < kColBatch; ++j) fw[j] = c[j] >= 0 ? __ldg(fb + (c[j] >> 5)) : ~0u;
            } else {
#pragma unroll
                for (int j = 0; j < kColBatch; ++j) fw[j] = 0u;
            }
#pragma unroll
            for (int j = 0; j < kColBatch; ++j) {
                if (c[j] < 0) continue;
                const int e = e0 + j * kThreads;
                MGNN_CHECK(o_tile + e < W.col_stride[hop] && c[j] < (W.remote ? W.n_global : pd.vp),
                           "cols o=%lld c=%d", o_tile + e, c[j]);
                cols[e] = c[j];
                const uint32_t bit = 1u << (c[j] & 31);
                if (!(fw[j] & bit)) atomicOr(&fb[c[j] >> 5], bit);
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ bitmap -> sorted new frontier nodes
// new_i = fb & ~fbp word by word (fb: every rank sampled so far, fbp: F_i); the popcount scan over
// words in rank order (= ascending id) appends new_i to the frontier (R#7) and writes, for EVERY
// word, the pair (new_i bits, frontier position of the word's first new node) that k_relabel reads;
// fbp catches up with fb for the next hop.
// Persistent: a block claims the instance's word tiles in order until they run out (kernel start-up
// -- PDL wait, constant loads -- was ~40 % of the stall samples with one short-lived block per tile).
__global__ void __launch_bounds__(kThreads, 8) k_compact(WinDev W, int hop, Scratch sc, int64_t tiles_max, int one_tile) {
    pdl_enter();
    __shared__ long long sm[8];
    __shared__ int tslot;
    __shared__ long long prefix_sh;
    __shared__ int32_t stage_sh[kCompactStage];  // the tile's new ranks in order (coalesced frontier writes)
    const int m = blockIdx.y;
    const PartDev& pd = W.parts[m / W.n_steps];
    const int64_t nwords = ((W.remote ? W.n_global : pd.vp) + 31) >> 5;   // rank space
    const int64_t ntiles = (nwords + kWordTile - 1) / kWordTile;
    uint32_t* nbp = W.nb + ((int64_t)m * W.L + hop) * W.bm_words * 2;   // word w: nbp[2w] bits, nbp[2w+1] position
    const uint32_t* fb = W.fb + (int64_t)m * W.bm_words;
    uint32_t* fbp = W.fbp + (int64_t)m * W.bm_words;
    int64_t* hs = W.hop_size + (int64_t)m * (kMaxLayers + 1);
    int32_t* fr = W.fr_rank + (int64_t)m * W.ucap;
    // arena bound of F_{hop+1} (mgnn_sampler_config_bounded): positions past it are not stored, the
    // size is clamped and the window is marked overflowed (every buffer-state kernel then skips it)
    const int64_t cap = hop + 1 < W.L ? W.off_stride[hop + 1] - 1 : W.ucap;
    for (int done = 0;; ++done) {
        if (one_tile && done) break;
        const int tile = claim_tile(sc.tilectr + m, &tslot);
        if (tile >= ntiles) break;
        const int64_t wd0 = (int64_t)tile * kWordTile + (int64_t)threadIdx.x * kCWords;   // 4 consecutive words
        uint32_t b[kCWords];
        uint4 now = make_uint4(0u, 0u, 0u, 0u);
        if (wd0 < nwords) {              // bm_words % kCWords == 0: one 16-byte load of each bitmap
            now = *reinterpret_cast<const uint4*>(fb + wd0);
            const uint4 was = *reinterpret_cast<const uint4*>(fbp + wd0);
            b[0] = now.x & ~was.x;
            b[1] = now.y & ~was.y;
            b[2] = now.z & ~was.z;
            b[3] = now.w & ~was.w;
        } else {
#pragma unroll
            for (int j = 0; j < kCWords; ++j) b[j] = 0u;
        }
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < kCWords; ++j) cnt += __popc(b[j]);
        long long agg;
        const long long excl = block_excl_scan256(cnt, sm, &agg);
        if (threadIdx.x < 32) {
            const unsigned long long pv = lookback_exclusive(sc.status + (int64_t)m * tiles_max, tile,
                                                             (unsigned long long)agg);
            if (threadIdx.x == 0) prefix_sh = (long long)pv;
        }
        __syncthreads();
        const int64_t nF = hs[hop];
        int64_t pos = nF + prefix_sh + excl;
        if (wd0 < nwords) {
            // new_i keeps its bitmap; with the word's first position it gives every new node's frontier
            // position as wpre + popc(lower bits) (k_relabel), without a scattered rank -> position table
            uint32_t p[kCWords];
            int64_t q = pos;
#pragma unroll
            for (int j = 0; j < kCWords; ++j) {
                p[j] = (uint32_t)q;
                q += __popc(b[j]);
            }
            uint4* v = reinterpret_cast<uint4*>(nbp + 2 * wd0);
            v[0] = make_uint4(b[0], p[0], b[1], p[1]);
            v[1] = make_uint4(b[2], p[2], b[3], p[3]);
            if (cnt) *reinterpret_cast<uint4*>(fbp + wd0) = now;
        }
        if (agg <= kCompactStage) {      // the tile's ranks go through shared memory, then out coalesced
            int q = (int)excl;
#pragma unroll
            for (int j = 0; j < kCWords; ++j) {
                const int64_t wd = wd0 + j;
                uint32_t bb = b[j];
                while (bb) {
                    const int bi = __ffs(bb) - 1;
                    bb &= bb - 1;
                    MGNN_CHECK(wd * 32 + bi < (W.remote ? W.n_global : pd.vp), "compact r=%lld", (long long)(wd * 32 + bi));
                    stage_sh[q++] = (int32_t)(wd * 32 + bi);
                }
            }
            __syncthreads();
            const int64_t base = nF + prefix_sh;
            for (int i = threadIdx.x; i < (int)agg; i += kThreads)
                if (base + i < cap) fr[base + i] = stage_sh[i];
        } else {
#pragma unroll
            for (int j = 0; j < kCWords; ++j) {
                const int64_t wd = wd0 + j;
                uint32_t bb = b[j];
                while (bb) {
                    const int bi = __ffs(bb) - 1;
                    bb &= bb - 1;
                    const int32_t r = (int32_t)(wd * 32 + bi);
                    MGNN_CHECK(r < (W.remote ? W.n_global : pd.vp), "compact r=%d", r);
                    if (pos < cap) fr[pos] = r;
                    ++pos;
                }
            }
        }
        if (tile == ntiles - 1 && threadIdx.x == 0) {
            const int64_t total = nF + prefix_sh + agg;
            hs[hop + 1] = total < cap ? total : cap;
            if (total > cap) atomicMin(W.ovf, (unsigned long long)W.step0);
        }
        __syncthreads();                 // prefix_sh / sm are reused by the next tile
    }
}

// ------------------------------------------------------------------ cols: rank -> position in F_{i+1}
// A sampled rank c of hop i is either a seed (position from k_seeds' table) or a new node of
// exactly one hop j <= i; then its position is wpre_j[c/32] + popc(new_j[c/32] & lower bits),
// since new_j is appended to the frontier in ascending rank order (R#7).
__device__ __forceinline__ int32_t frontier_pos(const WinDev& W, int m, int hop, const int2* __restrict__ sp,
                                                int32_t c, unsigned& probes) {
    const int64_t wd = c >> 5;
    const uint32_t bit = 1u << (c & 31);
    for (int j = hop; j >= 0; --j) {
        const int64_t o = ((int64_t)m * W.L + j) * W.bm_words + wd;
        const uint2 bp = __ldg(reinterpret_cast<const uint2*>(W.nb) + o);   // bits and position: one load
        ++probes;
        if (bp.x & bit) return (int32_t)bp.y + __popc(bp.x & (bit - 1u));
    }
    // a seed: its position in F_0 from the window's seed hash (k_seeds)
    for (uint32_t h = seed_hash(c) & (uint32_t)W.seed_hmask;; h = (h + 1) & (uint32_t)W.seed_hmask) {
        const int2 e = __ldg(sp + h);
        ++probes;
        if (e.x == c + 1) return e.y;
        if (e.x == 0) return 0;                  // not reached for a sampled column (overflowed window only)
    }
}

__global__ void __launch_bounds__(kThreads) k_relabel(WinDev W) {
    pdl_enter();
    const int m = blockIdx.y;
    const int2* sp = W.seedpos + (int64_t)m * (W.seed_hmask + 1);
    const int64_t* hs = W.hop_size + (int64_t)m * (kMaxLayers + 1);
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    if (W.sampled_units && blockIdx.x == 0 && threadIdx.x == 0) {   // roofline units (bench profiling)
        long long e = 0, f = 0;
        for (int hop = 0; hop < W.L; ++hop) {
            e += W.off[hop][(int64_t)m * W.off_stride[hop] + hs[hop]];
            f += hs[hop];
        }
        atomicAdd((unsigned long long*)&W.sampled_units[0], (unsigned long long)e);
        atomicAdd((unsigned long long*)&W.sampled_units[1], (unsigned long long)f);
        atomicAdd((unsigned long long*)&W.sampled_units[2], (unsigned long long)hs[W.L]);
    }
    unsigned probes = 0;                         // dependent probes (roofline units, profiling only)
    for (int hop = 0; hop < W.L; ++hop) {
        const int64_t* off = W.off[hop] + (int64_t)m * W.off_stride[hop];
        int32_t* cols = W.cols[hop] + (int64_t)m * W.col_stride[hop];
        const int64_t E = off[hs[hop]];
        const int32_t cap = (int32_t)hs[hop + 1];      // positions stay inside F_{hop+1} (clamped on overflow)
        // kRelabelBatch independent lookups in flight per thread (bitmap / prefix words are L2 reads)
        for (int64_t e0 = (int64_t)blockIdx.x * kThreads * kRelabelBatch + threadIdx.x; e0 < E;
             e0 += stride * kRelabelBatch) {
            int32_t c[kRelabelBatch];
#pragma unroll
            for (int j = 0; j < kRelabelBatch; ++j) c[j] = e0 + j * kThreads < E ? cols[e0 + j * kThreads] : 0;
#pragma unroll
            for (int j = 0; j < kRelabelBatch; ++j) {
                unsigned pr = 0;
                const int32_t p = frontier_pos(W, m, hop, sp, c[j], pr);
                if (e0 + j * kThreads < E) probes += pr;
                MGNN_CHECK(p >= 0 && (p < cap || *W.ovf <= W.step0 + (uint64_t)W.n_steps - 1 ||
                                      e0 + j * kThreads >= E),
                           "relabel pos=%d cap=%d", p, cap);
                c[j] = p < cap ? p : cap - 1;
            }
#pragma unroll
            for (int j = 0; j < kRelabelBatch; ++j)
                if (e0 + j * kThreads < E) cols[e0 + j * kThreads] = c[j];
        }
    }
    if (W.sampled_units) {
        for (int o = 16; o > 0; o >>= 1) probes += __shfl_xor_sync(kFull, probes, o);
        if ((threadIdx.x & 31) == 0 && probes) atomicAdd((unsigned long long*)&W.sampled_units[5], (unsigned long long)probes);
    }
}

// ------------------------------------------------------------------ launchers
void launch_seeds(const WinDev& w, cudaStream_t s) {
    dim3 grid(grid_x_for(w.batch, kThreads, w.n_inst), w.n_inst);
    launch_k(k_seeds, grid, dim3(kThreads), 0, s, w);
    count_launches(1, __func__, s);
}

void launch_hop(const WinDev& w, int hop, int64_t fcap, Scratch sc, cudaStream_t s) {
    // small hops (e.g. the seeds) use 64-node tiles so the launch still fills the GPU
    const char* te = getenv("MGNN_HOP_TILE");          // experiment: force the tile size
    const int T = te && atoi(te) == 64 ? 64 : ((fcap * (int64_t)w.n_inst) / 256 < (int64_t)num_sms() * 4 ? 64 : 256);
    const int64_t tiles_max = scan_tiles_count(fcap);          // scratch stride (64-node tiles)
    // persistent blocks (~5 resident per SM in total); each loops over claimed tiles
    int64_t tiles = (fcap + T - 1) / T;
    static const int grid_bps = [] {                 // resident-block cap of the persistent grid per SM
        const char* e = getenv("MGNN_HOP_GRID_BPS");  // (0 = one block per tile, not persistent)
        const int v = e ? atoi(e) : MGNN_HOP_BLOCKS;
        return v >= 0 && v <= 64 ? v : MGNN_HOP_BLOCKS;
    }();
    const int64_t target = ((int64_t)num_sms() * grid_bps + w.n_inst - 1) / w.n_inst;
    if (grid_bps > 0 && tiles > target) tiles = target;
    if (tiles < 1) tiles = 1;
    dim3 grid((unsigned)tiles, w.n_inst);
    ensure_smem_k(k_hop<uint64_t>, 256 * MGNN_MAX_FANOUT * 8);
    ensure_smem_k(k_hop<uint32_t>, 256 * MGNN_MAX_FANOUT * 4);
    const int64_t tm = tiles_max < 1 ? 1 : tiles_max;
    const char* f64 = getenv("MGNN_SAMPLE_IDX64");   // tests: force the 64-bit staging variant
    static const int align = [] {                    // 1: segment-aligned tiles across the window's instances
        const char* e = getenv("MGNN_HOP_ALIGN");
        return e ? atoi(e) : 0;
    }();
    static const int mark_filter = [] {              // 1: load the membership word before marking
        const char* e = getenv("MGNN_MARK_FILTER");  // (measured: products sampling 0.79 ms with 0,
        return e ? atoi(e) : 0;                      // 0.82 ms with 1; arxiv equal)
    }();
    if (w.idx32 && !(f64 && f64[0] == '1'))
        launch_k(k_hop<uint32_t>, grid, dim3(kThreads), (size_t)T * w.k_hop[hop] * 4, s, w, hop, sc, tm, T, mark_filter,
                 align, grid_bps == 0 && !align ? 1 : 0);
    else
        launch_k(k_hop<uint64_t>, grid, dim3(kThreads), (size_t)T * w.k_hop[hop] * 8, s, w, hop, sc, tm, T, mark_filter,
                 align, grid_bps == 0 && !align ? 1 : 0);
    count_launches(1, __func__, s);
}

void launch_compact(const WinDev& w, int hop, Scratch sc, cudaStream_t s) {
    const int64_t tiles = scan_tiles_words(w.bm_words);
    // persistent blocks: ~8 resident per SM over all instances, each looping over claimed tiles
    static const int per_sm = [] {
        const char* e = getenv("MGNN_COMPACT_BPS");
        const int v = e ? atoi(e) : 8;
        return v >= 0 && v <= 64 ? v : 8;            // 0: one block per tile (not persistent)
    }();
    int64_t gx = ((int64_t)num_sms() * per_sm + w.n_inst - 1) / w.n_inst;
    if (per_sm == 0 || gx > tiles) gx = tiles;
    dim3 grid((unsigned)(gx < 1 ? 1 : gx), w.n_inst);
    launch_k(k_compact, grid, dim3(kThreads), 0, s, w, hop, sc, (int64_t)(tiles < 1 ? 1 : tiles), per_sm == 0 ? 1 : 0);
    count_launches(1, __func__, s);
}

void launch_relabel(const WinDev& w, cudaStream_t s) {
    int64_t e_max = 0;
    for (int i = 0; i < w.L; ++i) e_max = w.col_stride[i] > e_max ? w.col_stride[i] : e_max;
    dim3 grid(grid_x_for(e_max, kThreads * kRelabelBatch, w.n_inst), w.n_inst);
    launch_k(k_relabel, grid, dim3(kThreads), 0, s, w);
    count_launches(1, __func__, s);
}

}  // namespace mgnn
