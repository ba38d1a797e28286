// gather.cu -- classify + feature gather (Alg.2 l.2-5, l.10-11, l.21-22).
//
// Every instance of the window at once (gridDim.y = instances).  A warp takes
// 32 consecutive nodes of F_L: lane i classifies node f0+i in parallel
//   local  (u in V_p^l)           -> row of the partition's own table   (l.10)
//   hit    (u in V_p^h, in BUF)   -> BUF row of its slot                 (l.11)
//   miss   (u in V_p^h, not BUF)  -> row of the OWNER's table, read over
//                                    NVLink peer memory when the owner is
//                                    another GPU (the RPC of l.22, fused into
//                                    the gather: no request/response exchange)
// -- a range test on the node's local rank plus one slot_of load (the compact
// O(|V_p^h|) S_A of P:228, indexed directly instead of by binary search) --
// then the warp copies the 32 rows with several 16-byte loads in flight per
// lane (source pointers broadcast by shuffles), so no row waits on the
// classification of the next.  Hits set bit w of the slot's hit mask (decay
// bookkeeping, l.6-9); misses add 1.0f to S_A (l.21): every operand is 1.0f,
// so the result does not depend on the order of the atomics.  X stores are
// streaming (evict-first) so the window's output does not flush the tables
// out of L2.
#include <algorithm>
#include <cstdlib>

#include "launch.h"

namespace mgnn {

constexpr int kGThreads = 256;
constexpr int kGWarps = kGThreads / 32;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void stcs4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }

// WIDE: rows of >= 32 float4 (D >= 128, one or more 16-B chunks per lane); else 32/q rows per warp step.
// Alg.2 l.2-5 for one frontier entry r: local row, buffer hit (hit recorded for the decay) or
// miss (S_A += 1, row from the owner's table -- over NVLink when it lives on another GPU).
// Returns the class 0 local, 1 hit, 2 miss, 4 miss from a peer GPU; sets the row and global id.
// Remote expansion (NEXT-1): ranks are global ids; nodes outside V_p^h are misses, not scored.
__device__ __forceinline__ int classify(const WinDev& W, const WorldDev& G, const PartDev& pd, int64_t r,
                                        unsigned long long wbit, const float*& src, int32_t& gid) {
    const int pitch = W.pitch;
    const int64_t rank_lo = W.remote ? pd.lo : pd.h_below;
    if (r >= rank_lo && r < rank_lo + pd.n_local) {
        gid = (int32_t)(pd.lo + (r - rank_lo));
        src = pd.table + (r - rank_lo) * pitch;
        return 0;
    }
    int64_t h;
    if (W.remote) {
        gid = (int32_t)r;
        h = pd.halo_map[r];
    } else {
        h = r < pd.h_below ? r : r - pd.n_local;
        gid = pd.halo_ids[h];
    }
    MGNN_CHECK(h < pd.n_h || W.remote, "classify h=%lld n_h=%lld", (long long)h, (long long)pd.n_h);
    if (h >= 0) {
        const int32_t s = pd.slot_of[h];
        MGNN_CHECK(s < pd.cap, "classify slot=%d cap=%lld", s, (long long)pd.cap);
        if (s >= 0) {
            src = pd.rows + (int64_t)s * pitch;
            atomicOr(&pd.hitmask[s], wbit);
            return 1;
        }
        atomicAdd(&pd.sa[h], 1.0f);
    }
    const int qo = owner_of(G.bounds, G.n_parts, gid);
    MGNN_CHECK(G.tables[qo] != nullptr && gid >= G.bounds[qo] && gid < G.bounds[qo + 1], "miss gid=%d owner=%d", gid,
               qo);
    src = G.tables[qo] + ((int64_t)gid - G.bounds[qo]) * pitch;
    return G.on_peer[qo] ? 4 : 2;
}

template <bool WIDE>
__global__ void __launch_bounds__(kGThreads, 4) k_gather(WinDev W, WorldDev G) {
    pdl_enter();
    if (*W.ovf <= W.step0 + (uint64_t)W.n_steps - 1) return;   // arena overflow: window skipped
    __shared__ unsigned long long cnt_sh[4];
    const int m = blockIdx.y;
    const int lp = m / W.n_steps, w = m % W.n_steps;
    const PartDev& pd = W.parts[lp];
    if (threadIdx.x < 4) cnt_sh[threadIdx.x] = 0;
    __syncthreads();
    const int64_t U = W.hop_size[(int64_t)m * (kMaxLayers + 1) + W.L];
    const int lane = threadIdx.x & 31;
    const int pitch = W.pitch;
    const int q = pitch >> 2;                      // float4 per row
    const int32_t* fr = W.fr_rank + (int64_t)m * W.ucap;
    int32_t* fgid = W.fr_gid + (int64_t)m * W.ucap;
    float* X = W.X + (int64_t)m * W.ucap * pitch;
    const unsigned long long wbit = 1ull << w;
    unsigned n_loc = 0, n_hit = 0, n_miss = 0, n_peer = 0;
    const int64_t stride = (int64_t)gridDim.x * kGWarps * 32;
    for (int64_t f0 = ((int64_t)blockIdx.x * kGWarps + (threadIdx.x >> 5)) * 32; f0 < U; f0 += stride) {
        // ---- classify 32 nodes, one per lane
        const int64_t f = f0 + lane;
        const bool valid = f < U;
        const float* src = nullptr;
        int cls = 3;
        if (valid) {
            int32_t gid;
            cls = classify(W, G, pd, fr[f], wbit, src, gid);
            fgid[f] = gid;
        }
        n_loc += __popc(__ballot_sync(kFull, cls == 0));
        n_hit += __popc(__ballot_sync(kFull, cls == 1));
        n_miss += __popc(__ballot_sync(kFull, cls >= 2 && cls != 3));
        n_peer += __popc(__ballot_sync(kFull, cls == 4));
        const int nrows = (int)(U - f0 < 32 ? U - f0 : 32);
        float* Xw = X + f0 * pitch;
        // ---- copy the rows, several independent 16-B loads in flight per lane
        if (WIDE) {
            constexpr int R = 8;                       // rows in flight per lane
            if (nrows == 32) {
#pragma unroll 1
                for (int j = 0; j < 32; j += R) {
                    const float* s[R];
#pragma unroll
                    for (int u = 0; u < R; ++u) s[u] = (const float*)__shfl_sync(kFull, (unsigned long long)src, j + u);
                    for (int c = lane * 4; c < pitch; c += 128) {
                        float4 v[R];
#pragma unroll
                        for (int u = 0; u < R; ++u) v[u] = ldg4(s[u] + c);
#pragma unroll
                        for (int u = 0; u < R; ++u) stcs4(Xw + (int64_t)(j + u) * pitch + c, v[u]);
                    }
                }
            } else {
                for (int j = 0; j < nrows; ++j) {
                    const float* s = (const float*)__shfl_sync(kFull, (unsigned long long)src, j);
                    for (int c = lane * 4; c < pitch; c += 128) stcs4(Xw + (int64_t)j * pitch + c, ldg4(s + c));
                }
            }
        } else {
            // q < 32 float4 per row: 32/q rows side by side per warp instruction
            const int per = 32 / q;
            const int sub = lane / q, ch = lane - sub * q;
            const bool act = sub < per;
            for (int j = 0; j < nrows; j += 4 * per) {
                float4 v[4];
                int row[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    row[u] = j + u * per + sub;
                    const float* s = (const float*)__shfl_sync(kFull, (unsigned long long)src, row[u] & 31);
                    if (act && row[u] < nrows) v[u] = ldg4(s + ch * 4);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (act && row[u] < nrows) stcs4(Xw + (int64_t)row[u] * pitch + ch * 4, v[u]);
            }
        }
    }
    if (lane == 0) {
        if (n_loc) atomicAdd(&cnt_sh[0], (unsigned long long)n_loc);
        if (n_hit) atomicAdd(&cnt_sh[1], (unsigned long long)n_hit);
        if (n_miss) atomicAdd(&cnt_sh[2], (unsigned long long)n_miss);
        if (n_peer) atomicAdd(&cnt_sh[3], (unsigned long long)n_peer);
    }
    __syncthreads();
    long long* cn = W.counts + (int64_t)m * 8;
    if (threadIdx.x == 0) {
        if (cnt_sh[0]) atomicAdd((unsigned long long*)&cn[1], cnt_sh[0]);
        if (cnt_sh[1]) atomicAdd((unsigned long long*)&cn[2], cnt_sh[1]);
        if (cnt_sh[2]) {
            atomicAdd((unsigned long long*)&cn[3], cnt_sh[2]);
            atomicAdd((unsigned long long*)&cn[6], cnt_sh[2]);
        }
        if (cnt_sh[3]) atomicAdd((unsigned long long*)&cn[7], cnt_sh[3]);
        const unsigned long long rows = cnt_sh[0] + cnt_sh[1] + cnt_sh[2];
        if (rows && W.gathered_rows) atomicAdd((unsigned long long*)W.gathered_rows, rows);
        if (W.prof_hm) {
            if (cnt_sh[1]) atomicAdd((unsigned long long*)&W.prof_hm[0], cnt_sh[1]);
            if (cnt_sh[2]) atomicAdd((unsigned long long*)&W.prof_hm[1], cnt_sh[2]);
        }
        if (blockIdx.x == 0) cn[0] = U;
    }
}

// ------------------------------------------------------------------ TMA bulk-copy variant
// Same classification; the rows move through shared memory with the copy engine instead of
// registers: per warp, two stages of R rows; lane j issues cp.async.bulk (global -> smem,
// completion counted on the stage's mbarrier) for row j of the next chunk while the current
// chunk's rows go out with cp.async.bulk smem -> global (bulk_group).  The SM keeps only the
// classification, so the concurrent sampling kernels get the issue slots and registers.
constexpr int kTWarps = 4;
constexpr int kTStageBytes = 8192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
// L2 policies: feature-table rows are re-read across the window (keep them), X rows are written
// once and read by the consumer later (let them go first).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_load_hint(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                               uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Work distribution: chunks of R consecutive rows of F_L are CLAIMED dynamically (one atomic per
// chunk on the instance's counter), so the kernel is work-conserving when its blocks start late --
// e.g. while the sampling kernels of the next window hold the SMs on the other stream.  A warp starts
// at its block's instance and moves on to the next instance once one is exhausted, until every
// instance is done; the counters are zeroed with the window (mgnn_sample).
__global__ void __launch_bounds__(kTWarps * 32) k_gather_tma(WinDev W, WorldDev G, int R, int stage_bytes, int hint,
                                                              int dyn) {
    pdl_enter();
    if (*W.ovf <= W.step0 + (uint64_t)W.n_steps - 1) return;   // arena overflow: window skipped
    extern __shared__ __align__(128) unsigned char tsm[];
    __shared__ __align__(8) uint64_t bars[kTWarps][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        mbar_init(&bars[warp][0], 1);
        mbar_init(&bars[warp][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int pitch = W.pitch;
    const uint32_t rowb = (uint32_t)pitch * 4u;
    unsigned char* stage[2] = {tsm + (size_t)warp * 2 * stage_bytes, tsm + (size_t)warp * 2 * stage_bytes + stage_bytes};
    uint32_t phase[2] = {0u, 0u};
    const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    // per-warp counters of the instance `acc_m`, flushed when the warp moves to another instance
    int acc_m = -1;
    unsigned n_loc = 0, n_hit = 0, n_miss = 0, n_peer = 0;
    auto flush = [&]() {
        if (acc_m >= 0 && lane == 0) {
            long long* cn = W.counts + (int64_t)acc_m * 8;
            if (n_loc) atomicAdd((unsigned long long*)&cn[1], (unsigned long long)n_loc);
            if (n_hit) atomicAdd((unsigned long long*)&cn[2], (unsigned long long)n_hit);
            if (n_miss) {
                atomicAdd((unsigned long long*)&cn[3], (unsigned long long)n_miss);
                atomicAdd((unsigned long long*)&cn[6], (unsigned long long)n_miss);
            }
            if (n_peer) atomicAdd((unsigned long long*)&cn[7], (unsigned long long)n_peer);
            const unsigned long long rows = (unsigned long long)n_loc + n_hit + n_miss;
            if (rows && W.gathered_rows) atomicAdd((unsigned long long*)W.gathered_rows, rows);
            if (W.prof_hm) {
                if (n_hit) atomicAdd((unsigned long long*)&W.prof_hm[0], (unsigned long long)n_hit);
                if (n_miss) atomicAdd((unsigned long long*)&W.prof_hm[1], (unsigned long long)n_miss);
            }
        }
        n_loc = n_hit = n_miss = n_peer = 0;
    };
    // claim the next chunk: instance m (advanced past exhausted instances), first row f0, its rows nr;
    // false = done
    int m = blockIdx.y, visited = 0;
    int64_t next_static = (int64_t)blockIdx.x * kTWarps + warp;      // dyn == 0 / 2: fixed chunk stride
    // dyn == 2 (segment-aligned chunks): F_L = F_0 ++ new_0 ++ ... ++ new_{L-1}, every segment sorted by
    // rank (R#7).  Chunk c of segment s covers the same FRACTION c / C_s of that segment in every instance
    // of the window (C_s = ceil(longest segment s / R)), so the instances, which the warps walk in lock
    // step, read the same rank region of the tables at the same time (L2 reuse across minibatches).
    __shared__ long long seg_c[kMaxLayers + 2];     // chunk prefix over segments (max over instances)
    if (dyn == 2) {
        if (threadIdx.x < kMaxLayers + 2) seg_c[threadIdx.x] = 0;
        __syncthreads();
        for (int mi = threadIdx.x; mi < W.n_inst; mi += blockDim.x) {
            const int64_t* hsi = W.hop_size + (int64_t)mi * (kMaxLayers + 1);
            for (int sgi = 0; sgi <= W.L; ++sgi) {
                const long long len = sgi == 0 ? hsi[0] : hsi[sgi] - hsi[sgi - 1];
                atomicMax(&seg_c[sgi + 1], (len + R - 1) / R);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int sgi = 1; sgi <= W.L + 1; ++sgi) seg_c[sgi] += seg_c[sgi - 1];
        __syncthreads();
    }
    int chunk_rows = R;
    auto claim = [&](int& cm, int64_t& f0) -> bool {
        if (dyn == 2) {
            const int64_t* hsm = W.hop_size + (int64_t)m * (kMaxLayers + 1);
            for (;;) {
                const int64_t j = next_static;
                next_static += (int64_t)gridDim.x * kTWarps;
                if (j >= seg_c[W.L + 1]) return false;
                int sgi = 0;
                while (j >= seg_c[sgi + 1]) ++sgi;
                const int64_t c = j - seg_c[sgi], C = seg_c[sgi + 1] - seg_c[sgi];
                const int64_t s0 = sgi == 0 ? 0 : hsm[sgi - 1], len = sgi == 0 ? hsm[0] : hsm[sgi] - hsm[sgi - 1];
                const int64_t a = s0 + c * len / C, b = s0 + (c + 1) * len / C;
                if (j == 0 && lane == 0) W.counts[(int64_t)m * 8] = hsm[W.L];
                if (b <= a) continue;
                cm = m;
                f0 = a;
                chunk_rows = (int)(b - a);
                return true;
            }
        }
        if (!dyn) {
            const int64_t U = W.hop_size[(int64_t)m * (kMaxLayers + 1) + W.L];
            const int64_t c = next_static;
            next_static += (int64_t)gridDim.x * kTWarps;
            if (c * R >= U) return false;
            if (c == 0 && lane == 0) W.counts[(int64_t)m * 8] = U;
            cm = m;
            f0 = c * R;
            return true;
        }
        while (visited < W.n_inst) {
            const int64_t U = W.hop_size[(int64_t)m * (kMaxLayers + 1) + W.L];
            int c = 0;
            if (lane == 0) c = atomicAdd(&W.gctr[m], 1);
            c = __shfl_sync(kFull, c, 0);
            if ((int64_t)c * R < U) {
                if (c == 0 && lane == 0) W.counts[(int64_t)m * 8] = U;     // |F_L| of the instance
                cm = m;
                f0 = (int64_t)c * R;
                return true;
            }
            m = m + 1 == W.n_inst ? 0 : m + 1;
            ++visited;
        }
        return false;
    };
    // classify chunk (cm, f0) (lanes < R) and issue its row loads into stage st; returns its rows
    auto issue = [&](int cm, int64_t f0, int st) -> int {
        if (cm != acc_m) {
            flush();
            acc_m = cm;
        }
        const int lp = cm / W.n_steps, w = cm % W.n_steps;
        const PartDev& pd = W.parts[lp];
        const int64_t U0 = W.hop_size[(int64_t)cm * (kMaxLayers + 1) + W.L];
        const int64_t U = dyn == 2 ? f0 + chunk_rows : U0;   // aligned chunks end inside F_L
        const int64_t f = f0 + lane;
        const bool valid = lane < R && f < U;
        const float* src = nullptr;
        int cls = 3;
        if (valid) {
            int32_t gid;
            cls = classify(W, G, pd, W.fr_rank[(int64_t)cm * W.ucap + f], 1ull << w, src, gid);
            W.fr_gid[(int64_t)cm * W.ucap + f] = gid;
        }
        n_loc += __popc(__ballot_sync(kFull, cls == 0));
        n_hit += __popc(__ballot_sync(kFull, cls == 1));
        n_miss += __popc(__ballot_sync(kFull, cls >= 2 && cls != 3));
        n_peer += __popc(__ballot_sync(kFull, cls == 4));
        const int nrows = (int)(U - f0 < R ? U - f0 : R);
        bulk_wait_read0();                       // stores that last read this stage are done
        __syncwarp();
        if (lane == 0) mbar_expect_tx(&bars[warp][st], (uint32_t)nrows * rowb);
        __syncwarp();
        if (valid) {
            if (hint & 1)
                bulk_load_hint(stage[st] + (size_t)lane * rowb, src, rowb, &bars[warp][st], pol_keep);
            else
                bulk_load(stage[st] + (size_t)lane * rowb, src, rowb, &bars[warp][st]);
        }
        return nrows;
    };
    int cm = 0, st = 0, nrows = 0;
    int64_t f0 = 0;
    bool have = claim(cm, f0);
    if (have) nrows = issue(cm, f0, st);
    while (have) {
        int nm = 0, nn = 0;
        int64_t fn = 0;
        const bool next = claim(nm, fn);
        if (next) nn = issue(nm, fn, st ^ 1);       // next chunk's loads overlap this chunk's wait
        mbar_wait(&bars[warp][st], phase[st]);
        phase[st] ^= 1u;
        float* X = W.X + ((int64_t)cm * W.ucap + f0) * pitch;
        if (hint & 8) {                          // stores through the LSU (smem -> registers -> X, streaming):
            // the copy engine then carries only the row reads (it is the per-SM limit of this kernel)
            const float4* s4 = reinterpret_cast<const float4*>(stage[st]);
            float4* x4 = reinterpret_cast<float4*>(X);
            const int n4 = (int)((uint32_t)nrows * rowb / 16u);
#pragma unroll 4
            for (int i = lane; i < n4; i += 32) __stcs(x4 + i, s4[i]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // reads done before the next TMA fill
            __syncwarp();
        } else if (hint & 4) {                   // the chunk's rows are contiguous in smem and in X:
            if (lane == 0) {                     // one bulk store of nrows rows
                if (hint & 2)
                    bulk_store_hint(X, stage[st], (uint32_t)nrows * rowb, pol_stream);
                else
                    bulk_store(X, stage[st], (uint32_t)nrows * rowb);
            }
        } else if (lane < nrows) {
            if (hint & 2)
                bulk_store_hint(X + (int64_t)lane * pitch, stage[st] + (size_t)lane * rowb, rowb, pol_stream);
            else
                bulk_store(X + (int64_t)lane * pitch, stage[st] + (size_t)lane * rowb, rowb);
        }
        bulk_commit();
        have = next;
        cm = nm;
        f0 = fn;
        nrows = nn;
        st ^= 1;
    }
    bulk_wait0();
    flush();
}

// ------------------------------------------------------------------ TMA row-gather variant (gather4)
// Same classification, but rows that come from a source on this GPU -- the partition's own table (local),
// its BUF rows (hits), or the table of another partition hosted by this context (misses) -- are loaded
// by the tensor-memory accelerator FOUR AT A TIME: a chunk of R rows (R % 4 == 0) is split into groups
// of 4 consecutive frontier positions; a group whose 4 rows share one source descriptor is one
// cp.async.bulk.tensor.2d...tile::gather4 (4 row indices, one instruction), any other row (mixed group,
// a peer GPU's table, the tail) one cp.async.bulk row copy as in k_gather_tma.  Frontier segments are
// sorted by rank (R#7), which keeps local rows and halo rows in runs, so most groups are pure.  Each
// group occupies a 128-byte-aligned slot of the stage and leaves with one bulk store (4 rows).
// Bulk copies take their operands from uniform registers, so a warp issues them one lane at a time:
// one instruction per 4 rows instead of one per row is what this variant buys.
__device__ __forceinline__ void g4_load(void* sdst, const void* map, int32_t r0, int32_t r1, int32_t r2, int32_t r3,
                                        uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(sdst)),
        "l"(map), "r"(smem_u32(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

__global__ void __launch_bounds__(kTWarps * 32) k_gather_g4(WinDev W, WorldDev G, const __grid_constant__ GatherMaps gm,
                                                             int R, int gstride, int hint) {
    pdl_enter();
    if (*W.ovf <= W.step0 + (uint64_t)W.n_steps - 1) return;   // arena overflow: window skipped
    extern __shared__ __align__(128) unsigned char tsm[];
    __shared__ __align__(8) uint64_t bars[kTWarps][2];
    __shared__ unsigned long long cnt_sh[4];
    const int m = blockIdx.y;
    const int lp = m / W.n_steps, w = m % W.n_steps;
    const PartDev& pd = W.parts[lp];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 4) cnt_sh[threadIdx.x] = 0;
    if (lane == 0) {
        mbar_init(&bars[warp][0], 1);
        mbar_init(&bars[warp][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int64_t U = W.hop_size[(int64_t)m * (kMaxLayers + 1) + W.L];
    const int pitch = W.pitch;
    const uint32_t rowb = (uint32_t)pitch * 4u;
    const int groups = R >> 2;
    const int stage_bytes = groups * gstride;
    const int32_t* fr = W.fr_rank + (int64_t)m * W.ucap;
    int32_t* fgid = W.fr_gid + (int64_t)m * W.ucap;
    float* X = W.X + (int64_t)m * W.ucap * pitch;
    unsigned char* base = tsm + ((128u - (smem_u32(tsm) & 127u)) & 127u);   // tensor copies: 128-B aligned
    unsigned char* stage[2] = {base + (size_t)warp * 2 * stage_bytes, base + (size_t)warp * 2 * stage_bytes + stage_bytes};
    const unsigned long long wbit = 1ull << w;
    const int n_lp = gm.n_lp;
    const int64_t rank_lo = W.remote ? pd.lo : pd.h_below;
    unsigned n_loc = 0, n_hit = 0, n_miss = 0, n_peer = 0;
    const int64_t stride = (int64_t)gridDim.x * kTWarps * R;
    uint32_t phase[2] = {0u, 0u};
    const uint64_t pol_stream = policy_evict_first();
    auto issue = [&](int64_t f0, int st) -> int {
        const int64_t f = f0 + lane;
        const bool valid = lane < R && f < U;
        const float* src = nullptr;
        int cls = 3, mid = -1;
        int32_t row = 0;
        if (valid) {
            int32_t gid;
            const int32_t r = fr[f];
            cls = classify(W, G, pd, r, wbit, src, gid);
            fgid[f] = gid;
            if (cls == 0) {                                   // own table
                mid = lp;
                row = (int32_t)(r - rank_lo);
            } else if (cls == 1) {                            // BUF slot
                mid = n_lp + lp;
                row = (int32_t)((src - pd.rows) / pitch);
            } else if (cls == 2) {                            // miss, owner on this GPU
                const int qo = owner_of(G.bounds, G.n_parts, gid);
                const int l2 = G.lp_of[qo];
                if (l2 >= 0) {
                    mid = l2;
                    row = (int32_t)(gid - G.bounds[qo]);
                }
            }
        }
        n_loc += __popc(__ballot_sync(kFull, cls == 0));
        n_hit += __popc(__ballot_sync(kFull, cls == 1));
        n_miss += __popc(__ballot_sync(kFull, cls >= 2 && cls != 3));
        n_peer += __popc(__ballot_sync(kFull, cls == 4));
        const int nrows = (int)(U - f0 < R ? U - f0 : R);
        // a group is pure when its 4 lanes are valid and share one descriptor
        const int g = lane >> 2, j = lane & 3;
        const int mid0 = __shfl_sync(kFull, mid, lane & ~3);
        const unsigned same = __ballot_sync(kFull, valid && mid >= 0 && mid == mid0);
        const bool pure = ((same >> (lane & ~3)) & 0xFu) == 0xFu;
        const int32_t r1 = __shfl_down_sync(kFull, row, 1), r2 = __shfl_down_sync(kFull, row, 2),
                      r3 = __shfl_down_sync(kFull, row, 3);
        bulk_wait_read0();                       // stores that last read this stage are done
        __syncwarp();
        if (lane == 0) mbar_expect_tx(&bars[warp][st], (uint32_t)nrows * rowb);
        __syncwarp();
        unsigned char* slot = stage[st] + (size_t)g * gstride;
        if (valid) {
            if (pure) {
                if (j == 0) g4_load(slot, &gm.maps[mid][0], row, r1, r2, r3, &bars[warp][st]);
            } else {
                bulk_load(slot + (size_t)j * rowb, src, rowb, &bars[warp][st]);
            }
        }
        return nrows;
    };
    int64_t f0 = ((int64_t)blockIdx.x * kTWarps + warp) * R;
    int st = 0;
    int nrows = f0 < U ? issue(f0, st) : 0;
    while (f0 < U) {
        const int64_t fn = f0 + stride;
        int nn = 0;
        if (fn < U) nn = issue(fn, st ^ 1);      // next chunk's loads overlap this chunk's wait
        mbar_wait(&bars[warp][st], phase[st]);
        phase[st] ^= 1u;
        const int gi = lane;                     // lane g stores group g (up to 4 rows)
        if (gi < groups && 4 * gi < nrows) {
            const int rows_g = nrows - 4 * gi < 4 ? nrows - 4 * gi : 4;
            float* dst = X + (f0 + 4 * gi) * pitch;
            const unsigned char* sg = stage[st] + (size_t)gi * gstride;
            if (hint & 2)
                bulk_store_hint(dst, sg, (uint32_t)rows_g * rowb, pol_stream);
            else
                bulk_store(dst, sg, (uint32_t)rows_g * rowb);
        }
        bulk_commit();
        f0 = fn;
        nrows = nn;
        st ^= 1;
    }
    bulk_wait0();
    if (lane == 0) {
        if (n_loc) atomicAdd(&cnt_sh[0], (unsigned long long)n_loc);
        if (n_hit) atomicAdd(&cnt_sh[1], (unsigned long long)n_hit);
        if (n_miss) atomicAdd(&cnt_sh[2], (unsigned long long)n_miss);
        if (n_peer) atomicAdd(&cnt_sh[3], (unsigned long long)n_peer);
    }
    __syncthreads();
    long long* cn = W.counts + (int64_t)m * 8;
    if (threadIdx.x == 0) {
        if (cnt_sh[0]) atomicAdd((unsigned long long*)&cn[1], cnt_sh[0]);
        if (cnt_sh[1]) atomicAdd((unsigned long long*)&cn[2], cnt_sh[1]);
        if (cnt_sh[2]) {
            atomicAdd((unsigned long long*)&cn[3], cnt_sh[2]);
            atomicAdd((unsigned long long*)&cn[6], cnt_sh[2]);
        }
        if (cnt_sh[3]) atomicAdd((unsigned long long*)&cn[7], cnt_sh[3]);
        const unsigned long long rows = cnt_sh[0] + cnt_sh[1] + cnt_sh[2];
        if (rows && W.gathered_rows) atomicAdd((unsigned long long*)W.gathered_rows, rows);
        if (W.prof_hm) {
            if (cnt_sh[1]) atomicAdd((unsigned long long*)&W.prof_hm[0], cnt_sh[1]);
            if (cnt_sh[2]) atomicAdd((unsigned long long*)&W.prof_hm[1], cnt_sh[2]);
        }
        if (blockIdx.x == 0) cn[0] = U;
    }
}

// ------------------------------------------------------------------ flat register variant
// Same classification; a warp's chunk of R <= 32 consecutive frontier rows is copied as ONE flat run
// of nrows * q float4 (q = pitch / 4): lane l moves elements l, l + 32, l + 64, ... so every load and
// store instruction is fully active whatever q is (a 100-d row is 25 float4: the per-row loop of
// k_gather leaves 7 of 32 lanes idle), UNR 16-byte loads are in flight per lane, and the X stores of
// the chunk are contiguous.  No shared-memory staging: the sampling kernels of the next window can be
// resident beside it.  Chunks are segment-aligned as in k_gather_tma (dyn == 2).
constexpr int kFThreads = 256;
constexpr int kFWarps = kFThreads / 32;
template <int kFUnroll, int kMinBlocks>
__global__ void __launch_bounds__(kFThreads, kMinBlocks) k_gather_flat(WinDev W, WorldDev G) {
    pdl_enter();
    if (*W.ovf <= W.step0 + (uint64_t)W.n_steps - 1) return;   // arena overflow: window skipped
    __shared__ unsigned long long cnt_sh[4];
    __shared__ long long seg_c[kMaxLayers + 2];
    const int m = blockIdx.y;
    const int lp = m / W.n_steps, w = m % W.n_steps;
    const PartDev& pd = W.parts[lp];
    const int64_t* hsm = W.hop_size + (int64_t)m * (kMaxLayers + 1);
    const int R = 32;
    if (threadIdx.x < 4) cnt_sh[threadIdx.x] = 0;
    if (threadIdx.x < kMaxLayers + 2) seg_c[threadIdx.x] = 0;
    __syncthreads();
    // chunk c of segment s covers the same fraction of that segment in every instance (see k_gather_tma)
    for (int mi = threadIdx.x; mi < W.n_inst; mi += blockDim.x) {
        const int64_t* hsi = W.hop_size + (int64_t)mi * (kMaxLayers + 1);
        for (int sgi = 0; sgi <= W.L; ++sgi) {
            const long long len = sgi == 0 ? hsi[0] : hsi[sgi] - hsi[sgi - 1];
            atomicMax(&seg_c[sgi + 1], (len + R - 1) / R);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int sgi = 1; sgi <= W.L + 1; ++sgi) seg_c[sgi] += seg_c[sgi - 1];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pitch = W.pitch;
    const int q = pitch >> 2;
    const unsigned long long wbit = 1ull << w;
    const int32_t* fr = W.fr_rank + (int64_t)m * W.ucap;
    int32_t* fgid = W.fr_gid + (int64_t)m * W.ucap;
    float4* X4 = reinterpret_cast<float4*>(W.X + (int64_t)m * W.ucap * pitch);
    unsigned n_loc = 0, n_hit = 0, n_miss = 0, n_peer = 0;
    const int64_t nchunks = seg_c[W.L + 1];
    for (int64_t j = (int64_t)blockIdx.x * kFWarps + warp; j < nchunks; j += (int64_t)gridDim.x * kFWarps) {
        int sgi = 0;
        while (j >= seg_c[sgi + 1]) ++sgi;
        const int64_t c = j - seg_c[sgi], C = seg_c[sgi + 1] - seg_c[sgi];
        const int64_t s0 = sgi == 0 ? 0 : hsm[sgi - 1], len = sgi == 0 ? hsm[0] : hsm[sgi] - hsm[sgi - 1];
        const int64_t a = s0 + c * len / C, b = s0 + (c + 1) * len / C;
        if (b <= a) continue;
        const int nrows = (int)(b - a);
        // ---- classify the chunk's rows, one per lane
        const float* src = nullptr;
        int cls = 3;
        if (lane < nrows) {
            int32_t gid;
            cls = classify(W, G, pd, fr[a + lane], wbit, src, gid);
            fgid[a + lane] = gid;
        }
        n_loc += __popc(__ballot_sync(kFull, cls == 0));
        n_hit += __popc(__ballot_sync(kFull, cls == 1));
        n_miss += __popc(__ballot_sync(kFull, cls >= 2 && cls != 3));
        n_peer += __popc(__ballot_sync(kFull, cls == 4));
        // ---- flat copy: element e = row (e / q), column (e % q); rows of the chunk are contiguous in X
        const int total = nrows * q;
        float4* Xc = X4 + a * q;
        int row = lane / q, col = lane - row * q;           // element `lane`, advanced by 32 per step
        const int drow = 32 / q, dcol = 32 - drow * q;
        for (int e0 = 0; e0 < total; e0 += 32 * kFUnroll) {
            float4 v[kFUnroll];
            int rr = row, cc = col;
#pragma unroll
            for (int u = 0; u < kFUnroll; ++u) {
                const float4* sp = reinterpret_cast<const float4*>(
                    __shfl_sync(kFull, (unsigned long long)src, rr & 31));
                if (e0 + u * 32 + lane < total) v[u] = __ldg(sp + cc);
                rr += drow;
                cc += dcol;
                if (cc >= q) {
                    cc -= q;
                    ++rr;
                }
            }
#pragma unroll
            for (int u = 0; u < kFUnroll; ++u)
                if (e0 + u * 32 + lane < total) __stcs(Xc + e0 + u * 32 + lane, v[u]);
            row = rr;
            col = cc;
        }
    }
    if (lane == 0) {
        if (n_loc) atomicAdd(&cnt_sh[0], (unsigned long long)n_loc);
        if (n_hit) atomicAdd(&cnt_sh[1], (unsigned long long)n_hit);
        if (n_miss) atomicAdd(&cnt_sh[2], (unsigned long long)n_miss);
        if (n_peer) atomicAdd(&cnt_sh[3], (unsigned long long)n_peer);
    }
    __syncthreads();
    long long* cn = W.counts + (int64_t)m * 8;
    if (threadIdx.x == 0) {
        if (cnt_sh[0]) atomicAdd((unsigned long long*)&cn[1], cnt_sh[0]);
        if (cnt_sh[1]) atomicAdd((unsigned long long*)&cn[2], cnt_sh[1]);
        if (cnt_sh[2]) {
            atomicAdd((unsigned long long*)&cn[3], cnt_sh[2]);
            atomicAdd((unsigned long long*)&cn[6], cnt_sh[2]);
        }
        if (cnt_sh[3]) atomicAdd((unsigned long long*)&cn[7], cnt_sh[3]);
        const unsigned long long rows = cnt_sh[0] + cnt_sh[1] + cnt_sh[2];
        if (rows && W.gathered_rows) atomicAdd((unsigned long long*)W.gathered_rows, rows);
        if (W.prof_hm) {
            if (cnt_sh[1]) atomicAdd((unsigned long long*)&W.prof_hm[0], cnt_sh[1]);
            if (cnt_sh[2]) atomicAdd((unsigned long long*)&W.prof_hm[1], cnt_sh[2]);
        }
        if (blockIdx.x == 0) cn[0] = hsm[W.L];
    }
}

void launch_gather(const WinDev& w, const WorldDev& world, bool l2_resident, const GatherMaps* g4, cudaStream_t s) {
    // exactly one wave of 4 resident 256-thread blocks per SM in total (64 registers per thread):
    // floor, so no second, nearly empty wave leaves SMs idle at the tail
    int64_t target = ((int64_t)num_sms() * 4) / w.n_inst;
    int64_t need = (w.ucap + kGWarps * 32 - 1) / (kGWarps * 32);
    unsigned gx = (unsigned)(need < target ? need : target);
    if (gx < 1) gx = 1;
    // MGNN_GATHER: flat (default) = k_gather_flat; tma = TMA bulk copies (k_gather_tma, or k_gather_g4 when
    // the hosted tables fit in L2); reg = the per-row register gather of round 1.  Pipelined windows
    // (tools/exp_window.py, sampling of the next window beside the gather, profiles/r02/gather_flat/):
    // products 2.01 -> 1.91 ms, reddit 2.27 -> 2.03, papers_s32 2.05 -> 1.99, arxiv 0.220 -> 0.211, cfg1
    // equal.  Alone the flat gather is slower on products (1.24 vs 1.14 ms) -- the TMA variants hold
    // 192 KB of staging per SM, so the sampling kernels cannot be resident beside them.
    static const int use_tma = [] {
        const char* e = getenv("MGNN_GATHER");
        return e && e[0] == 't' ? 1 : 0;
    }();
    static const bool use_flat = [] {
        const char* e = getenv("MGNN_GATHER");
        return !(e && (e[0] == 't' || e[0] == 'r'));
    }();
    static const int flat_bps = [] {
        const char* e = getenv("MGNN_FLAT_BPS");
        const int v = e ? atoi(e) : 0;
        return v >= 1 && v <= 256 ? v : 4;
    }();
    if (use_flat) {
        const int64_t tgt = std::max<int64_t>(1, ((int64_t)num_sms() * flat_bps) / w.n_inst);
        const int64_t nd = (w.ucap + kFWarps * 32 - 1) / (kFWarps * 32);
        const unsigned gxf = (unsigned)std::max<int64_t>(1, std::min(nd, tgt));
        static const int flat_unr = [] {
            const char* e = getenv("MGNN_FLAT_UNR");
            return e ? atoi(e) : 4;
        }();
        const dim3 gf(gxf, w.n_inst), bf(kFThreads);
        // the measured variants (profiles/r02/gather_flat/exp_s10*, all parity-tested); > 6 blocks per
        // SM: more, shorter blocks of <4, 4>
        switch ((flat_bps > 6 ? 4 : flat_bps) * 16 + flat_unr) {
            case 3 * 16 + 8: launch_k(k_gather_flat<8, 3>, gf, bf, 0, s, w, world); break;
            case 3 * 16 + 6: launch_k(k_gather_flat<6, 3>, gf, bf, 0, s, w, world); break;
            case 4 * 16 + 6: launch_k(k_gather_flat<6, 4>, gf, bf, 0, s, w, world); break;
            case 5 * 16 + 2: launch_k(k_gather_flat<2, 5>, gf, bf, 0, s, w, world); break;
            case 4 * 16 + 2: launch_k(k_gather_flat<2, 4>, gf, bf, 0, s, w, world); break;
            default: launch_k(k_gather_flat<4, 4>, gf, bf, 0, s, w, world); break;
        }
        count_launches(1, __func__, s);
        return;
    }
    // staging per warp: 2 stages of `stage` bytes; `bps` resident blocks per SM (one wave).  The
    // shared memory left on each SM is what the concurrently running sampling kernels can use.
    // 192 KB of staging per SM either way.  When the gathered tables fit in L2 (reads hit L2, the
    // X writes are the DRAM traffic) 4 KB stages x 6 blocks per SM keep more warps issuing: +3 % on
    // arxiv; from DRAM, 8 KB x 3 wins (products -13 %, papers_s32 -8 % with the small stages).
    static const int stage_env = [] {
        const char* e = getenv("MGNN_GATHER_STAGE");
        const int v = e ? atoi(e) : 0;
        return v >= 1024 && v <= 32768 ? v : 0;
    }();
    static const int bps_env = [] {
        const char* e = getenv("MGNN_GATHER_BPS");
        const int v = e ? atoi(e) : 0;
        return v >= 1 && v <= 8 ? v : 0;
    }();
    const bool small = l2_resident && (int64_t)w.pitch * 4 <= 1024;
    const int stage = stage_env ? stage_env : (small ? kTStageBytes / 2 : kTStageBytes);
    const int bps = bps_env ? bps_env : (small ? 6 : 3);
    const int R = (int)std::min<int64_t>(32, std::max<int64_t>(1, stage / ((int64_t)w.pitch * 4)));
    // row gather (gather4): 1 = always, 0 = never, 2 (default) = when the hosted tables fit in L2.
    // Measured: arxiv (L2-resident) 0.228 -> 0.214 ms per pipelined window; products (from DRAM) gather
    // alone 1.256 -> 1.297 ms and the pipelined window 2.22 -> 2.63 ms, so DRAM-bound gathers keep the
    // per-row copies.
    static const int use_g4 = [] {
        const char* e = getenv("MGNN_GATHER_G4");
        return e ? atoi(e) : 2;
    }();
    if (use_tma && (use_g4 == 1 || (use_g4 == 2 && l2_resident)) && g4 && w.feat_dim == w.pitch && w.pitch <= 256) {
        // R rows per chunk (a multiple of 4), each group of 4 in a 128-byte-aligned slot
        const int gstride = (int)(((int64_t)4 * w.pitch * 4 + 127) / 128 * 128);
        const int groups = std::max(1, std::min(8, (stage + gstride / 2) / gstride));
        const int Rg = 4 * groups;
        const size_t smem = (size_t)kTWarps * 2 * groups * gstride + 128;
        ensure_smem_k(k_gather_g4, (int)smem);
        int64_t tgt = ((int64_t)num_sms() * bps) / w.n_inst;
        int64_t nd = (w.ucap + kTWarps * Rg - 1) / (kTWarps * Rg);
        unsigned gxt = (unsigned)std::max<int64_t>(1, std::min(nd, tgt));
        static const int hint = [] {
            const char* e = getenv("MGNN_GATHER_HINT");
            return e ? atoi(e) & 7 : 6;
        }();
        launch_k(k_gather_g4, dim3(gxt, w.n_inst), dim3(kTWarps * 32), smem, s, w, world, *g4, Rg, gstride, hint);
    } else if (use_tma && (int64_t)w.pitch * 4 <= stage) {
        const size_t smem = (size_t)kTWarps * 2 * stage;
        ensure_smem_k(k_gather_tma, (int)smem);
        int64_t tgt = ((int64_t)num_sms() * bps) / w.n_inst;
        int64_t nd = (w.ucap + kTWarps * R - 1) / (kTWarps * R);
        unsigned gxt = (unsigned)std::max<int64_t>(1, std::min(nd, tgt));
        // L2 hints: 2 (default) = X rows stored evict_first, so the once-written minibatch does not push
        // the re-read feature tables and CSR out of L2 (+1-2 % on arxiv / products / papers_s32);
        // 1 = table rows loaded evict_last (alone: -3 % on arxiv), 3 = both, 0 = none
        // 4 = one bulk store per chunk instead of one per row (default 2 | 4: products pipelined window
        // 2.295 -> 2.254 ms, arxiv 0.238 -> 0.228 ms; products gather alone 1.197 -> 1.257 ms)
        static const int hint = [] {
            const char* e = getenv("MGNN_GATHER_HINT");
            return e ? atoi(e) & 7 : 6;
        }();
        // chunk assignment: 2 (default) = segment-aligned fixed stride (products gather alone 1.254 ->
        // 1.148 ms: the window's instances read the same rank region together; pipelined window equal);
        // 0 = fixed stride over F_L; 1 = dynamic claiming (one atomic per chunk; measured slower: 1.19 ->
        // 1.51 ms, the claim is on the issue path)
        static const int dyn = [] {
            const char* e = getenv("MGNN_GATHER_DYN");
            return e ? atoi(e) : 2;
        }();
        launch_k(k_gather_tma, dim3(gxt, w.n_inst), dim3(kTWarps * 32), smem, s, w, world, R, stage, hint, dyn);
    } else {
        dim3 grid(gx, w.n_inst);
        if (w.pitch >= 128)
            launch_k(k_gather<true>, grid, dim3(kGThreads), 0, s, w, world);
        else
            launch_k(k_gather<false>, grid, dim3(kGThreads), 0, s, w, world);
    }
    count_launches(1, __func__, s);
}

}  // namespace mgnn
