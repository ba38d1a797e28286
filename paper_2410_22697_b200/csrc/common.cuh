// common.cuh -- shared device types and primitives of the mgnn CUDA library
// (B200 / sm_100a).  Nothing here is shared with oracle/ (independent code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#ifndef MGNN_MAX_LAYERS
#define MGNN_MAX_LAYERS 8
#endif
#ifndef MGNN_MAX_FANOUT
#define MGNN_MAX_FANOUT 32
#endif

// Device bounds checks, compiled in with -DMGNN_CHECKS (debug builds only).
#ifdef MGNN_CHECKS
#define MGNN_CHECK(cond, fmt, ...)                                                            \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("[mgnn check] %s:%d " fmt "\n", __FILE__, __LINE__, __VA_ARGS__);          \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define MGNN_CHECK(cond, fmt, ...) \
    do {                           \
    } while (0)
#endif

namespace mgnn {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ Philox4x32-10
// Counter-based RNG (Salmon et al. SC'11) for every random draw (DESIGN R#4).
struct u4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u4 philox4x32_10(u4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = u4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Philox stream ids (the low byte of counter word 3; R#4).
constexpr uint32_t kStreamSample = 1, kStreamShuffle = 2, kStreamFeature = 3;

// ------------------------------------------------------------------ per-partition device state
struct PartDev {
    int32_t part_id;
    int64_t lo;          // V_p^l = [lo, lo + n_local)
    int64_t n_local;
    int64_t n_h;         // |V_p^h|
    int64_t h_below;     // halo ids < lo; local rank space: [0,h_below) halo, [h_below, h_below+n_local) local, rest halo
    int64_t vp;          // n_local + n_h
    int64_t n_train;
    int64_t cap;         // |BUF|
    int64_t nbatch;      // minibatches per epoch = ceil(n_train / B) (R#8)
    int32_t perm_slots;  // epoch orders kept resident (ring)
    const int64_t* indptr;     // [n_local+1]
    const int32_t* cols_rank;  // [nnz] neighbour ranks
    const int32_t* halo_ids;   // [n_h] ascending
    const int32_t* deg_in;     // [n_h]
    const int32_t* train_ids;  // [n_train] ascending
    const float* table;        // [n_local][pitch] own feature table
    // prefetcher state
    float* rows;               // [cap][pitch] BUF rows
    float* se;                 // [cap] S_E by slot
    float* sa;                 // [n_h] S_A by halo index
    int32_t* slot_of;          // [n_h] slot or -1
    int32_t* slot_h;           // [cap] halo index in slot
    unsigned long long* hitmask;  // [cap] bit w = hit at window step w
    int32_t* rank_deg;         // [n_h] position in the (deg_in desc, id asc) order (replacement tie-break)
    int32_t* deg_order;        // [n_h] halo index at each position of that order (inverse of rank_deg)
    int32_t* perm;             // [perm_slots][n_train] epoch orders
    const int32_t* halo_map;   // [n_global] halo index or -1 (remote expansion only)
};

// Global (graph-wide) read-only view: every partition's table (local or peer-mapped).
struct WorldDev {
    int32_t n_parts;
    int32_t pitch;
    const int64_t* bounds;      // [P+1]
    const float* const* tables; // [P] device-accessible pointers (NVLink peer pointers for remote)
    const uint8_t* on_peer;     // [P] 1 if the table lives on another GPU (rows cross NVLink)
    const int8_t* lp_of;        // [P] local index of partition q in this context, or -1
};

__device__ __forceinline__ int owner_of(const int64_t* __restrict__ bounds, int P, int64_t v) {
    int lo = 0, hi = P;  // find q with bounds[q] <= v < bounds[q+1]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (bounds[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

// rank -> global id inside partition pd
__device__ __forceinline__ int32_t rank_to_gid(const PartDev& pd, int32_t r) {
    if (r < pd.h_below) return pd.halo_ids[r];
    if (r < pd.h_below + pd.n_local) return (int32_t)(pd.lo + (r - pd.h_below));
    return pd.halo_ids[r - pd.n_local];
}

// ------------------------------------------------------------------ decoupled look-back
// Tile status word: [63:62] flag (0 none, 1 aggregate, 2 inclusive prefix), [61:0] value.
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by ALL 32 lanes of one warp of tile `tile` with the tile's aggregate;
// returns (to every lane) the exclusive prefix of all earlier tiles of the
// same segment.  The warp inspects 32 predecessors per round (one status load
// per lane), so a chain of published aggregates costs one L2 round trip per 32
// tiles instead of one per tile.  status[] must be zero before the launch;
// tiles are claimed in order (dynamic tile ids), so every waited-on
// predecessor is already resident.
__device__ __forceinline__ unsigned long long lookback_exclusive(unsigned long long* status, int tile,
                                                                 unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_status(&status[0], kFlagInc | agg);
        return 0;
    }
    if (lane == 0) st_status(&status[tile], kFlagAgg | agg);
    unsigned long long excl = 0;
    int base = tile - 1;                       // lane l looks at tile base - l
    while (true) {
        const int j = base - lane;
        const unsigned long long s = j >= 0 ? ld_status(&status[j]) : kFlagInc;
        const unsigned long long f = s & ~kValMask;
        const unsigned inc = __ballot_sync(kFull, f == kFlagInc);
        const unsigned none = __ballot_sync(kFull, f == 0);
        const int first = inc ? __ffs(inc) - 1 : 31;          // nearest inclusive predecessor
        const unsigned need = first == 31 ? kFull : ((2u << first) - 1u);
        if (none & need) continue;             // a needed predecessor has not published yet
        unsigned long long v = lane <= first ? (s & kValMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        excl += v;
        if (inc) break;
        base -= 32;
    }
    if (lane == 0) st_status(&status[tile], kFlagInc | (excl + agg));
    return excl;
}

// Block-wide exclusive scan of one long long per thread (blockDim.x == 256).
// Returns the thread's exclusive prefix; *total receives the block sum.
// smem must hold 8 long longs.  Contains __syncthreads.
__device__ __forceinline__ long long block_excl_scan256(long long v, long long* smem, long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem[warp] = x;
    __syncthreads();
    long long wpre = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        long long s = smem[i];
        if (i < warp) wpre += s;
        tot += s;
    }
    __syncthreads();
    *total = tot;
    return wpre + x - v;
}

// Programmatic dependent launch: a kernel launched with programmatic stream serialization is
// set up while its predecessor in the stream drains and waits here, before touching any memory
// the predecessor produces or consumes (a no-op for a normal launch).  Kernels do not trigger
// their successors early: waiting blocks would hold SM slots the concurrent stream needs
// (measured: +7% with the implicit trigger at exit, -2% with an early trigger).
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Dynamic, in-order tile id for a segment (claimed by thread 0, broadcast).
__device__ __forceinline__ int claim_tile(int32_t* ctr, int* smem_slot) {
    if (threadIdx.x == 0) *smem_slot = atomicAdd(ctr, 1);
    __syncthreads();
    int t = *smem_slot;
    return t;
}

}  // namespace mgnn
